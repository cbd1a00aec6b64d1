C1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C1 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_dyn -s 3 -c 1 -o gpurun_out/prof_sweep_final_r01 $C1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
