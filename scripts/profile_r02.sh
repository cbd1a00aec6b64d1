#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): the bench line, its ncu launch list, and
# ncu --set full captures of the fused sweep (config 2), the cluster IMGS at k ~ 150 (config 2
# recipe) and the single-CTA IMGS + the small-M sweep on config 1 -- each capture after a plain
# run of the same command.  Outputs in gpurun_out/ (copied to profiles/r02/ by hand).
set -x
B="python bench.py --steps 20 --warmup 5"
$B > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
C1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C1 > gpurun_out/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $C1 > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep_dyn -s 3 -c 1 -o gpurun_out/prof_sweep_r02 $C1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
C2="python bench.py --steps 160 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_imgs -s 150 -c 1 -o gpurun_out/prof_imgs_r02 $C2 > gpurun_out/ncu3.log 2>&1; echo ncu3 rc=$?
C3="python scripts/run_config.py 1"
$C3 > gpurun_out/plain4.log 2>&1 && RBG_NO_DEVICE_LOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1_r02.csv $C3 > gpurun_out/ncu4.log 2>&1; echo ncu4 rc=$?
RBG_NO_DEVICE_LOOP=1 ncu --set full --clock-control none --import-source on -k regex:k_imgs_cta -s 40 -c 1 -o gpurun_out/prof_imgs_cta_r02 $C3 > gpurun_out/ncu5.log 2>&1; echo ncu5 rc=$?
RBG_NO_DEVICE_LOOP=1 ncu --set full --clock-control none --import-source on -k regex:k_sweep_dyn -s 40 -c 1 -o gpurun_out/prof_sweep_cfg1_r02 $C3 > gpurun_out/ncu6.log 2>&1; echo ncu6 rc=$?
