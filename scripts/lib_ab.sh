#!/bin/bash
# A/B of two builds of librbg.so on one box: paper_1805_06124_b200/librbg_old.so (baseline) vs
# the current librbg.so, alternated; $@ = the command to time (e.g. python scripts/imgs_scaling.py)
P=paper_1805_06124_b200
cp $P/librbg.so /tmp/librbg_new.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/librbg_new.so $P/librbg.so; else cp $P/librbg_old.so $P/librbg.so; fi
    echo "== $v (rep $rep)"; "$@" 2>&1 | tail -${AB_TAIL:-4}
  done
done
cp /tmp/librbg_new.so $P/librbg.so
