#!/bin/bash
# Block Jacobi evidence: phase trace (RBG_DEBUG_JACOBI) and one ncu --set full capture with source.
RBG_DEBUG_JACOBI=1 python scripts/recon_probe.py --reps 2 > gpurun_out/jac_trace.txt 2>&1; echo trace rc=$?
python scripts/recon_probe.py --reps 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bjacobi -c 1 -o gpurun_out/prof_bjacobi python scripts/recon_probe.py --reps 1 > gpurun_out/ncu_jac.log 2>&1; echo ncu rc=$?
