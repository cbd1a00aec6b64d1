#!/bin/bash
# Last-wave L2 prefetch A/B (RBG_LASTWAVE_PF = waves of columns prefetched at claim time).
python scripts/env_ab_probe.py RBG_LASTWAVE_PF 0 1 2 > gpurun_out/lastwave_small.jsonl 2> gpurun_out/lastwave_small.err; echo small rc=$?
RBG_LASTWAVE_PF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/lastwave_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/lastwave_parity.log
