#!/bin/bash
# After the scratch pool / pinned outputs: the GPU suite, then CUPTI traces of the NEXT-row calls.
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_scratch.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_scratch.log
for c in eim reconstruct gram; do python scripts/api_trace.py --call $c --out /tmp/$c.json > gpurun_out/api_trace2_$c.json 2>/dev/null; echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/api_trace2_$c.json')); print('$c wall_ms', [round(x*1e3,2) for x in d['walls_s']], 'gpu_busy_ms', round(d['gpu_busy_us']/1e3,2), {k: v for k, v in list(d['runtime_calls'].items())[:5]})"; done
python scripts/bench_next.py > gpurun_out/bench_next_scratch.json 2> gpurun_out/bench_next_scratch.err; echo next rc=$?
