#!/bin/bash
# Runs the GPU parity suites (hot path, validation/enrichment, EIM) once per library switch of
# every variant must give the oracle's bits.  Usage (on a B200):
#   bash scripts/check_switches.sh
set -u
cd "$(dirname "$0")/.."
for v in "RBG_SWEEP_KIND=percol" "RBG_IMGS_PRE=0" "RBG_IMGS_CTAS=8" "RBG_IMGS_BULK=1" "RBG_NO_PDL=1" "RBG_NO_TAIL_PF=1" "RBG_NO_DEVICE_LOOP=1" \
         "RBG_SWEEP_UNROLL=8" "RBG_COEFF=passes" "RBG_COEFF_CFG=2x6" "RBG_EIM=block" "RBG_EIM=warp1" "RBG_EIM_RESID=w" "RBG_IMGS_SMALL=0"; do
    echo "== $v"
    env "$v" timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_validation.py tests/test_eim.py \
        -q -m gpu -x 2>&1 | tail -1
done
