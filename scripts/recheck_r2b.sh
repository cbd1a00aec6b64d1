set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2b.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/smoke_r2b.log
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2b.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_r2b.log
timeout 900 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?
cat gpurun_out/bench_r2b.json
