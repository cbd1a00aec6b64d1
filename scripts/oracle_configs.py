#!/usr/bin/env python
"""CPU oracle timings on configs 0 and 1 (SURVEY §8(d) "Oracle timing": all host cores and one
thread, per-iteration wall time, it/s, effective sweep GB/s; nproc, CPU model, RAM), to sit
beside the GPU whole-greedy timings of scripts/bench_configs.py.  The oracle runs as it
stands (canonical lanes), on the same seeded inputs.  Prints one JSON line per run."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1805_06124_b200 import inputs  # noqa: E402


def host():
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        ram = [l for l in open("/proc/meminfo") if l.startswith("MemTotal")][0].split()[1]
        ram_gb = int(ram) / 1e6
    except OSError:
        ram_gb = None
    return {"nproc": len(os.sched_getaffinity(0)), "cpu_model": model, "ram_gb": ram_gb}


def main():
    h = host()
    cases = [("config0", inputs.config0()), ("config1", inputs.config1())]
    for name, (S, w, tol, k_max) in cases:
        M, N = S.shape
        se = 16 if S.dtype.kind == "c" else 8
        for threads in (h["nproc"], 1):   # explicit: omp_set_num_threads persists in the process
            t0 = time.perf_counter()
            r = O.greedy(S, w, tol, k_max, threads=threads)
            dt = time.perf_counter() - t0
            sweeps = r.k + 1
            out = {"config": name, "shape": [N, M], "threads": threads, "k": int(r.k),
                   "stop": r.stop, "s_total": dt, "ms_per_iter": dt / max(r.k, 1) * 1e3,
                   "iters_per_s": r.k / dt, "sweep_GBps": sweeps * N * M * se / dt / 1e9, **h}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
