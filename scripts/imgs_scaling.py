"""Per-iteration IMGS time vs k on the chirp workload (reduced M), from the library's events.

    python scripts/imgs_scaling.py [cols] [k_max]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 40960
K = int(sys.argv[2]) if len(sys.argv) > 2 else 300
ORTHO = sys.argv[3] if len(sys.argv) > 3 else "mgs"
N = 10000
t = inputs.chirp_grid(N)
w = inputs.simpson_weights(N)
q, chi, psi = inputs.chirp_params(M, 2, spin=True)
S = torch.empty((M, N), dtype=torch.complex128, device="cuda")
rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
ctx = rbg.Context(S, w, 0.0, K, ortho=ORTHO)
ctx.set_timing(True)
ctx.run()
k = ctx.info()[0]
sw, xc, im = ctx.timings(k)
nu = ctx.nu()
print(f"k={k}  sweep avg {np.nanmean(sw):.3f} ms  imgs avg {np.mean(im):.3f} ms  nu counts {np.bincount(nu)}")
for i in [1, 2, 5, 10, 25, 50, 100, 150, 200, 250, k - 1]:
    if i < k:
        steps = max(nu[i] * i, 1)
        print(f"k={i:4d} nu={nu[i]} imgs {im[i] * 1e3:8.1f} us  per MGS step {im[i] * 1e3 / steps:6.3f} us")
ctx.close()
