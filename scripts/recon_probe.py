#!/usr/bin/env python
"""Reconstruction probe (DESIGN.md f-3): a k-vector config-2-shaped greedy on --cols columns,
then ctx.reconstruct() timed (wall of the blocking call); RBG_DEBUG_JACOBI=1 prints the block
Jacobi's per-phase round times and sweep count."""
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
    p.add_argument("--cols", type=int, default=40960)
    p.add_argument("--k", type=int, default=300)
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    N = 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(a.cols, 2, spin=True)
    S = torch.empty((a.cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
    with rbg.Context(S, w, 0.0, a.k) as ctx:
        ctx.run()
        ts, tg = [], []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.gram()
            tg.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            sigma, kr, X = ctx.reconstruct(1e-3)
            ts.append(time.perf_counter() - t0)
    print(json.dumps({"k": a.k, "gram_s": min(tg), "reconstruct_s": min(ts), "kr": int(kr)}), flush=True)


if __name__ == "__main__":
    main()
