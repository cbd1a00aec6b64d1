#!/bin/bash
# EIM after a solver change: parity (bit-exact nodes / B vs the oracle, canaries), wall, warm launch list.
timeout 900 python -m pytest tests/test_eim.py tests/test_gpu_canary.py -q -x > gpurun_out/eim_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/eim_parity.log
RBG_EIM=warp1 timeout 900 python -m pytest tests/test_eim.py -q -x > gpurun_out/eim_parity_warp1.log 2>&1; echo parity_warp1 rc=$?; tail -1 gpurun_out/eim_parity_warp1.log
for rep in 1 2; do python scripts/api_trace.py --out /tmp/t.json > gpurun_out/eim_trace_s.$rep.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/eim_trace_s.$rep.json')); print('wall_ms', round(min(d['walls_s'])*1e3,2), 'gpu_busy_ms', round(d['gpu_busy_us']/1e3,2), 'span_ms', round(d['gpu_span_us']/1e3,2))"; done
python scripts/eim_probe.py --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:eim --csv --log-file gpurun_out/eim_s_launches.csv python scripts/eim_probe.py --reps 1 > gpurun_out/ncu_eim_s.log 2>&1; echo ncu rc=$?
