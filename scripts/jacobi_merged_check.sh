#!/bin/bash
# Block Jacobi with the merged tile update (default) vs the split passes (RBG_JACOBI_SPLIT=1).
timeout 900 python -m pytest tests/test_reconstruction.py tests/test_gpu_canary.py tests/test_gpu_scratch.py -q -x > gpurun_out/jm_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/jm_parity.log
RBG_JACOBI_SPLIT=1 timeout 900 python -m pytest tests/test_reconstruction.py -q -x 2>&1 | tail -1
RBG_DEBUG_JACOBI=1 python scripts/recon_probe.py --reps 2 > gpurun_out/jm_trace.txt 2>&1; grep -E 'round [1-3]:|sweeps=|max off' gpurun_out/jm_trace.txt | head -5
for rep in 1 2; do for v in merged split; do
  if [ $v = split ]; then export RBG_JACOBI_SPLIT=1; else unset RBG_JACOBI_SPLIT; fi
  python scripts/api_trace.py --call reconstruct --out /tmp/r.json > gpurun_out/jm_$v.$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/jm_$v.$rep.json')); print('$v', 'wall_ms', [round(x*1e3,2) for x in d['walls_s']], 'gpu_busy_ms', round(d['gpu_busy_us']/1e3,2))"
done; done
unset RBG_JACOBI_SPLIT
python scripts/recon_probe.py --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:'k_bjacobi|k_gram|k_recon|k_eig' --csv --log-file gpurun_out/recon_launches_merged.csv python scripts/recon_probe.py --reps 1 > /dev/null 2>&1; echo ncu rc=$?
