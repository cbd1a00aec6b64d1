#!/bin/bash
# Block Jacobi after a change: reconstruction parity (tolerance vs LAPACK eigh, Gram bit-exact), canaries,
# the phase trace and the wall of rbg_reconstruct.
timeout 900 python -m pytest tests/test_reconstruction.py tests/test_gpu_canary.py -q -x > gpurun_out/jac_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/jac_parity.log
RBG_DEBUG_JACOBI=1 python scripts/recon_probe.py --reps 2 > gpurun_out/jac_trace2.txt 2>&1; echo trace rc=$?
grep -E 'round [1-3]:|sweeps=|max off' gpurun_out/jac_trace2.txt | head -6; tail -1 gpurun_out/jac_trace2.txt
python scripts/recon_probe.py --reps 3 > gpurun_out/jac_wall.json 2>&1; cat gpurun_out/jac_wall.json
python scripts/recon_probe.py --reps 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:'k_bjacobi|k_gram|k_recon|k_eig' --csv --log-file gpurun_out/recon_launches.csv python scripts/recon_probe.py --reps 1 > gpurun_out/ncu_recon.log 2>&1; echo ncu rc=$?
