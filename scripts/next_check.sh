#!/bin/bash
# NEXT rows after a change: EIM parity (all modes) + canaries, warm launch list of the EIM kernels,
# and CUPTI traces of the blocking eim / reconstruct / gram calls (wall vs GPU time vs host calls).
timeout 900 python -m pytest tests/test_eim.py tests/test_gpu_canary.py tests/test_reconstruction.py -q -x > gpurun_out/next_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/next_parity.log
for v in "RBG_EIM=warp1" "RBG_EIM=block" "RBG_EIM_RESID=w"; do env "$v" timeout 600 python -m pytest tests/test_eim.py -q -x 2>&1 | tail -1; done
for c in eim reconstruct gram; do python scripts/api_trace.py --call $c --out /tmp/$c.json > gpurun_out/api_trace_$c.json 2>/dev/null; echo "$c rc=$?"; cat gpurun_out/api_trace_$c.json; done
python scripts/eim_probe.py --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:eim --csv --log-file gpurun_out/eim_s3_launches.csv python scripts/eim_probe.py --reps 1 > gpurun_out/ncu_eim_s3.log 2>&1; echo ncu rc=$?
