#!/bin/bash
# Scratch pool on / off (RBG_NO_SCRATCH) in one build, alternated: validate sequence and bench_next.
for rep in 1 2; do for v in on off; do
  if [ $v = off ]; then export RBG_NO_SCRATCH=1; else unset RBG_NO_SCRATCH; fi
  echo "== $v (rep $rep)"; python scripts/validate_probe.py 409600 2>&1 | tail -5
done; done
for v in on off; do
  if [ $v = off ]; then export RBG_NO_SCRATCH=1; else unset RBG_NO_SCRATCH; fi
  python scripts/bench_next.py > gpurun_out/bench_next_ab2_$v.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_next_ab2_$v.json').read().strip().splitlines()[-1])
print('$v validate', round(d['validate']['s']*1e3,1), 'reconstruct', round(d['reconstruct']['total_s']*1e3,2), 'eim', round(d['eim']['s']*1e3,2), 'add', round(d['add_columns_4096_s']*1e3,1), round(d['add_columns_4096_again_s']*1e3,1))"
done
