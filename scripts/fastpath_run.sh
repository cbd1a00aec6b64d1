#!/bin/bash
# A/B: the sweep's predicate-free path for whole groups (fast) against the previous build (base).
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/fast_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/fast_parity.log
export AB_TAIL=1
LIBS="base fast" bash scripts/libs_ab.sh python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/fast_ab_bench.txt 2>&1; echo ab rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/fast_ab_bench.txt"):
    if l.startswith("=="): tag=l.strip(); continue
    try: d=json.loads(l)
    except Exception: continue
    print(tag, round(d["value"],2), "sweep", round(d["phase_ms_avg"]["sweep"],4), "GB/s", round(d["roofline"]["achieved"]), "SM", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
LIBS="base fast" AB_TAIL=17 bash scripts/libs_ab.sh python scripts/imgs_probe_r2.py ab > gpurun_out/fast_ab_small.txt 2>&1; echo small rc=$?
