# ncu --set full of the 16-CTA IMGS kernel at k ~ 150 (cfg2 workload), then the exchange probe
C2="python bench.py --steps 160 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/plain_imgs.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_imgs -s 150 -c 1 -o gpurun_out/prof_imgs_c16 $C2 > gpurun_out/ncu_imgs.log 2>&1; echo ncu rc=$?
timeout 600 python scripts/xchg_probe.py > gpurun_out/xchg_probe.txt 2>&1; cat gpurun_out/xchg_probe.txt
