set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
C2="python bench.py --steps 200 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_imgs -s 150 -c 1 -o gpurun_out/prof_imgs_b $C2 > gpurun_out/ncu3.log 2>&1; echo ncu3 rc=$?
C1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C1 > gpurun_out/plain1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 -o gpurun_out/prof_sweep_b $C1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
