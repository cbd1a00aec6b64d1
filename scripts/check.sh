# usage: bash scripts/check.sh [bench args...]  -- GPU tests then one bench run
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print({k: l.get(k) for k in ['value','ms_per_step','phase_ms_avg','hbm_gbs_per_gpu']}, l['roofline']['frac'], l.get('e2e',{}).get('value'), l['clocks'])"
