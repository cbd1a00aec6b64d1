# sweep variants (RBG_SWEEP_KIND = percol | ring | tma) on the cfg2 workload; GPU tests; full bench
for V in ${VARIANTS:-ring tma}; do
 for U in ${UNROLLS:-12}; do
  RBG_SWEEP_KIND=$V RBG_SWEEP_UNROLL=$U timeout 300 python bench.py --steps ${STEPS:-40} --warmup 3 --no-e2e --no-cpu > gpurun_out/tune_${V}_U$U.log 2>&1
  python -c "import json;l=json.loads(open('gpurun_out/tune_${V}_U$U.log').read().strip().splitlines()[-1]);print('$V U=$U', round(l['value'],2), round(l['roofline']['achieved'],1), l['phase_ms_avg'], l['clocks']['sm_mhz'])" || tail -5 gpurun_out/tune_${V}_U$U.log
 done
done
if [ -n "$TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
fi
if [ -n "$FULL" ]; then
timeout 900 python bench.py $FULL_ARGS > gpurun_out/bench_full.log 2>&1; echo full rc=$?
tail -1 gpurun_out/bench_full.log
fi
