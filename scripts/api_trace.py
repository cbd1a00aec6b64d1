#!/usr/bin/env python
"""Where the wall time of a NEXT-row call goes: torch.profiler (CUPTI) trace of one ctx.eim() /
ctx.reconstruct() / ctx.gram() call (--call) on a k-vector config-2-shaped basis -- GPU kernel
time, the gaps between kernels, and the runtime API calls on the host (cudaLaunchKernel,
cudaMalloc, cudaMemcpy, ...)."""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cols", type=int, default=20480)
    p.add_argument("--k", type=int, default=300)
    p.add_argument("--out", default="gpurun_out/eim_trace.json")
    p.add_argument("--call", default="eim", choices=["eim", "reconstruct", "gram", "validate"])
    p.add_argument("--val-cols", type=int, default=40960)
    a = p.parse_args()
    N = 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(a.cols, 2, spin=True)
    S = torch.empty((a.cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
    with rbg.Context(S, w, 0.0, a.k) as ctx:
        ctx.run()
        V = None
        if a.call == "validate":
            qv, cv, pv = inputs.chirp_params(a.val_cols, 12, spin=True)
            V = torch.empty((a.val_cols, N), dtype=torch.complex128, device="cuda")
            rbg.gen_chirp(V, t, w, qv, cv, pv, spin=True)
        call = {"eim": ctx.eim, "reconstruct": lambda: ctx.reconstruct(1e-3), "gram": ctx.gram,
                "validate": lambda: ctx.validate(V)}[a.call]
        call()
        torch.cuda.synchronize()
        walls = []
        for _ in range(2):
            t0 = time.perf_counter()
            call()
            walls.append(time.perf_counter() - t0)
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            t0 = time.perf_counter()
            call()
            wall = time.perf_counter() - t0
    prof.export_chrome_trace(a.out)
    ev = json.load(open(a.out))["traceEvents"]
    kern = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
    rt = [e for e in ev if e.get("cat") == "cuda_runtime" or e.get("cat") == "cuda_driver"]
    busy = sum(e["dur"] for e in kern)
    span = (kern[-1]["ts"] + kern[-1]["dur"] - kern[0]["ts"]) if kern else 0
    agg = {}
    for e in rt:
        d = agg.setdefault(e["name"], [0, 0.0])
        d[0] += 1
        d[1] += e["dur"]
    print(json.dumps({"walls_s": walls, "profiled_wall_s": wall, "kernels": len(kern), "gpu_busy_us": busy,
                      "gpu_span_us": span,
                      "runtime_calls": {k: {"n": v[0], "total_us": round(v[1], 1)} for k, v in
                                        sorted(agg.items(), key=lambda x: -x[1][1])[:12]}}), flush=True)


if __name__ == "__main__":
    main()
