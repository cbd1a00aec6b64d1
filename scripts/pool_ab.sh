#!/bin/bash
# A/B of the scratch-pool build against the previous one: validate sequence and bench_next.
export AB_TAIL=6
LIBS="base pool" bash scripts/libs_ab.sh python scripts/validate_probe.py 409600 > gpurun_out/pool_ab_validate.txt 2>&1; echo ab rc=$?
cat gpurun_out/pool_ab_validate.txt
for v in base pool; do cp paper_1805_06124_b200/librbg_$v.so paper_1805_06124_b200/librbg.so; python scripts/bench_next.py > gpurun_out/bench_next_ab_$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_next_ab_$v.json').read().strip().splitlines()[-1])
print('$v validate', round(d['validate']['s']*1e3,1), 'reconstruct', round(d['reconstruct']['total_s']*1e3,2), 'eim', round(d['eim']['s']*1e3,2), 'add', round(d['add_columns_4096_s']*1e3,1), round(d['add_columns_4096_again_s']*1e3,1))"; done
cp paper_1805_06124_b200/librbg_pool.so paper_1805_06124_b200/librbg.so
