#!/bin/bash
# Round-2 checkpoint on one B200 (under gpurun): the whole GPU suite, the bench line (default
# and --steps 20), IMGS vs k, and an ncu --set full capture of the cluster IMGS at k ~ 150 after
# a plain run of the same command.  Outputs in gpurun_out/ (copied to profiles/r02/ by hand).
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ckpt.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_ckpt.log
python bench.py > gpurun_out/bench_ckpt_default.json 2> gpurun_out/bench_ckpt_default.err; echo bench rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ckpt_20.json 2> gpurun_out/bench_ckpt_20.err; echo bench20 rc=$?
python scripts/imgs_scaling.py 40960 300 > gpurun_out/imgs_scaling_ckpt.txt 2>&1; echo scaling rc=$?
C2="python bench.py --steps 160 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/plain_imgs.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_imgs -s 150 -c 1 -o gpurun_out/prof_imgs_r02b $C2 > gpurun_out/ncu_imgs.log 2>&1; echo ncu rc=$?
