#!/bin/bash
# A/B of several builds of librbg.so on one box: LIBS="base v1 ..." names
# paper_1805_06124_b200/librbg_<name>.so files, alternated twice; $@ = the command to time.
P=paper_1805_06124_b200
cp $P/librbg.so /tmp/librbg_current.so
for rep in 1 2; do
  for v in $LIBS; do
    cp $P/librbg_$v.so $P/librbg.so
    echo "== $v (rep $rep)"; "$@" 2>&1 | tail -${AB_TAIL:-4}
  done
done
cp /tmp/librbg_current.so $P/librbg.so
