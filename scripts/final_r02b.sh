#!/bin/bash
# Last-session final evidence on one B200 (under gpurun): smoke, the whole GPU suite, every library
# switch through the parity suites, the bench line (default and --steps 20) and its ncu launch list.
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final_b.log 2>&1; echo smoke rc=$?
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final_b.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu_final_b.log
bash scripts/check_switches.sh > gpurun_out/check_switches_final_b.txt 2>&1; echo switches rc=$?
cat gpurun_out/check_switches_final_b.txt
python bench.py > gpurun_out/bench_final_b_default.json 2> gpurun_out/bench_final_b_default.err; echo bench rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final_b_20.json 2> gpurun_out/bench_final_b_20.err; echo bench20 rc=$?
C1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C1 > gpurun_out/plain1_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_b.csv $C1 > gpurun_out/ncu1_b.log 2>&1; echo ncu1 rc=$?
python scripts/api_trace.py --out /tmp/e.json > gpurun_out/eim_trace_final_b.json 2>/dev/null; echo eim rc=$?
python scripts/bench_next.py > gpurun_out/bench_next_final_b.json 2> gpurun_out/bench_next_final_b.err; echo next rc=$?
