# ncu evidence for the final round-1 build: the bench launch list and one --set full capture
# of the sweep (4th launch) and of IMGS at k ~ 150, each after a plain run of the same command
set -x
C1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C1 > gpurun_out/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_r01.csv $C1 > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
$C1 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_dyn -s 3 -c 1 -o gpurun_out/prof_sweep_final_r01 $C1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
C2="python bench.py --steps 160 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_imgs -s 150 -c 1 -o gpurun_out/prof_imgs_final_r01 $C2 > gpurun_out/ncu3.log 2>&1; echo ncu3 rc=$?
