#!/bin/bash
# EIM residual: TMA-staged tiles (default) vs per-thread load rings (RBG_EIM_RESID=w), parity + A/B.
timeout 900 python -m pytest tests/test_eim.py tests/test_gpu_canary.py -q -x > gpurun_out/eim_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/eim_parity.log
for rep in 1 2; do
  python scripts/api_trace.py --out /tmp/t.json > gpurun_out/eim_trace_t.$rep.json 2>/dev/null; echo t rc=$?
  RBG_EIM_RESID=w python scripts/api_trace.py --out /tmp/w.json > gpurun_out/eim_trace_w.$rep.json 2>/dev/null; echo w rc=$?
done
for f in gpurun_out/eim_trace_[tw].*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', 'wall_ms', round(min(d['walls_s'])*1e3,2), 'gpu_busy_ms', round(d['gpu_busy_us']/1e3,2), 'span_ms', round(d['gpu_span_us']/1e3,2))"; done
python scripts/eim_probe.py --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:eim --csv --log-file gpurun_out/eim_t_launches.csv python scripts/eim_probe.py --reps 1 > gpurun_out/ncu_eim_t.log 2>&1; echo ncu rc=$?
python scripts/eim_probe.py --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_eim_residual_t -s 150 -c 1 -o gpurun_out/prof_eim_resid_t python scripts/eim_probe.py --reps 1 > gpurun_out/ncu_eim_t2.log 2>&1; echo ncu2 rc=$?
