#!/bin/bash
# EIM: wall of rbg_eim (k = 300) and a warm-cache ncu launch list (--cache-control none) of one call.
python scripts/eim_probe.py --reps 3 > gpurun_out/eim_wall.json 2>&1; echo wall rc=$?; cat gpurun_out/eim_wall.json
python scripts/eim_probe.py --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:eim --csv --log-file gpurun_out/eim_warm_launches.csv python scripts/eim_probe.py --reps 1 > gpurun_out/ncu_eim.log 2>&1; echo ncu rc=$?
