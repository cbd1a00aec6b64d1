#!/usr/bin/env python
"""EIM probe (DESIGN.md f-2): a k-vector config-2-shaped basis from a greedy on --cols columns,
then ctx.eim() timed (wall of the blocking call) for the default warp-level kernels and for
RBG_EIM=block.  Small enough for an ncu launch list."""
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
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    N = 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(a.cols, 2, spin=True)
    S = torch.empty((a.cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
    out = {}
    with rbg.Context(S, w, 0.0, a.k) as ctx:
        ctx.run()
        for mode in ("warp", "block"):
            if mode == "block":
                os.environ["RBG_EIM"] = "block"
            ts = []
            for _ in range(a.reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                nodes, _ = ctx.eim()
                ts.append(time.perf_counter() - t0)
            os.environ.pop("RBG_EIM", None)
            out[mode] = {"s": min(ts), "us_per_step": min(ts) / len(nodes) * 1e6, "k": len(nodes)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
