set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
for U in 4 8 12 16; do
  RBG_SWEEP_UNROLL=$U timeout 300 python bench.py --cols-per-gpu 204800 --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/tune_U$U.log 2>&1
  python -c "import json;l=json.loads(open('gpurun_out/tune_U$U.log').read().strip().splitlines()[-1]);print('U=$U', l['roofline']['achieved'], l['phase_ms_avg'], l['clocks'])"
done
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo full rc=$?
tail -1 gpurun_out/bench_full.log
