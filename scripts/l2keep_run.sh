#!/bin/bash
# L2-resident prefix A/B (scripts/l2keep_probe.py) + config-2 bench with and without it.
python scripts/env_ab_probe.py RBG_L2_KEEP_MB 0 32 64 96 > gpurun_out/l2keep_small.jsonl 2> gpurun_out/l2keep_small.err; echo small rc=$?
for rep in 1 2; do for mb in 0 48; do
RBG_L2_KEEP_MB=$mb python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/l2keep_bench_$mb.$rep.json 2>/dev/null; echo bench $mb rc=$?
python - <<PY
import json; d=json.load(open("gpurun_out/l2keep_bench_$mb.$rep.json")); print("$mb", d["value"], d["phase_ms_avg"], d["clocks"]["sm_mhz"])
PY
done; done
RBG_L2_KEEP_MB=64 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/l2keep_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/l2keep_parity.log
