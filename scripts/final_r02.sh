#!/bin/bash
# Round-2 final evidence on one B200 (under gpurun): the whole GPU suite, the opt-in config-3
# two-shard test, the bench line (default and --steps 20), its ncu launch list, and --set full
# captures of the sweep and the cluster IMGS, each after a plain run of the same command.
# Outputs in gpurun_out/ (copied to profiles/r02/ by hand).
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu_final.log
RBG_FULLSIZE_ORACLE=1 timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -k whole_oracle > gpurun_out/fullsize_cfg3_final.log 2>&1; echo cfg3 rc=$?
tail -2 gpurun_out/fullsize_cfg3_final.log
python bench.py > gpurun_out/bench_final_default.json 2> gpurun_out/bench_final_default.err; echo bench rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final_20.json 2> gpurun_out/bench_final_20.err; echo bench20 rc=$?
C1="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C1 > gpurun_out/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $C1 > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep_dyn -s 3 -c 1 -o gpurun_out/prof_sweep_final $C1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
