#!/bin/bash
# Closing check of the last session on one B200: smoke, the whole GPU suite, the default bench line.
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final_c.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_final_c.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final_c.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_final_c.log
python bench.py > gpurun_out/bench_final_c.json 2> gpurun_out/bench_final_c.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_final_c.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'])"
