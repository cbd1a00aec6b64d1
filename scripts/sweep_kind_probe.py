"""Per-launch sweep time vs column count for the load-ring variants (RBG_SWEEP_KIND env is
read per launch): validation passes (rbg_validate = sweep 0 + k coefficient sweeps) on
blocks of M columns against a k = 20 basis.

    python scripts/sweep_kind_probe.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

N, K = 10000, 20
t = inputs.chirp_grid(N)
w = inputs.simpson_weights(N)
q, chi, psi = inputs.chirp_params(40960, 2, spin=True)
S = torch.empty((40960, N), dtype=torch.complex128, device="cuda")
rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
ctx = rbg.Context(S, w, 0.0, K)
ctx.run()
for M in (4096, 40960, 204800):
    qv, cv, pv = inputs.chirp_params(M, 12, spin=True)
    V = torch.empty((M, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(V, t, w, qv, cv, pv, spin=True)
    for kind in ("percol", "ring", "percol", "ring"):
        os.environ["RBG_SWEEP_KIND"] = kind
        ctx.validate(V[:256])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.validate(V)
        dt = time.perf_counter() - t0
        gb = (K + 1) * M * N * 16 / 1e9
        print(f"M={M:7d} {kind:7s} {dt * 1e3:8.2f} ms  {gb / dt:8.1f} GB/s (incl. upload copy + NaN scan)", flush=True)
    del V
    torch.cuda.empty_cache()
