#!/usr/bin/env python
"""Blocked coefficient kernel probe (coeff.cu): a k-vector config-2-shaped basis from a greedy
on --cols columns, then validate() of --val-cols independent chirp columns, timed (CUDA events
around the blocking call) for the blocked kernel and for RBG_COEFF=passes.  Small enough for ncu:
    ncu -k regex:k_coeff_block -c 1 --set full python scripts/coeff_probe.py --reps 1
"""
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
    p.add_argument("--val-cols", type=int, default=40960)
    p.add_argument("--k", type=int, default=300)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--passes", action="store_true")
    a = p.parse_args()
    N = 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(a.cols, 2, spin=True)
    S = torch.empty((a.cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
    qv, cv, pv = inputs.chirp_params(a.val_cols, 12, spin=True)
    V = torch.empty((a.val_cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(V, t, w, qv, cv, pv, spin=True)
    out = {}
    with rbg.Context(S, w, 0.0, a.k) as ctx:
        ctx.run()
        k = ctx.result(full=False).k
        for mode in (["block", "passes"] if a.passes else ["block"]):
            if mode == "passes":
                os.environ["RBG_COEFF"] = "passes"
            ts = []
            for _ in range(a.reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ctx.validate(V)
                ts.append(time.perf_counter() - t0)
            os.environ.pop("RBG_COEFF", None)
            tb = min(ts)
            out[mode] = {"s": tb, "TFLOPs": 8.0 * k * a.val_cols * N / tb / 1e12}
    out["k"] = k
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
