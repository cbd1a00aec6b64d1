#!/bin/bash
# EIM with programmatic dependent launches between the step kernels vs without (RBG_NO_PDL).
timeout 900 python -m pytest tests/test_eim.py tests/test_gpu_scratch.py -q -x > gpurun_out/eim_pdl_parity.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/eim_pdl_parity.log
RBG_NO_PDL=1 timeout 900 python -m pytest tests/test_eim.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in pdl nopdl; do
  if [ $v = nopdl ]; then export RBG_NO_PDL=1; else unset RBG_NO_PDL; fi
  python scripts/api_trace.py --call eim --out /tmp/e.json > gpurun_out/eim_pdl_$v.$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/eim_pdl_$v.$rep.json')); print('$v', 'wall_ms', [round(x*1e3,2) for x in d['walls_s']], 'gpu_busy_ms', round(d['gpu_busy_us']/1e3,2), 'span_ms', round(d['gpu_span_us']/1e3,2))"
done; done
