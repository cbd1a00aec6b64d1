#!/usr/bin/env python
"""Phase timestamps of one IMGS launch (RBG_DEBUG_IMGS=<iteration> is read per context):
    python scripts/imgs_trace_r2.py <iteration> [timing 0|1] [cols]
prints the library's stderr lines (per-phase %globaltimer and, if k >= 64, MGS step cycles)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

it = int(sys.argv[1])
timing = len(sys.argv) > 2 and sys.argv[2] == "1"
M = int(sys.argv[3]) if len(sys.argv) > 3 else 40960
cfg = int(sys.argv[4]) if len(sys.argv) > 4 else 2       # 2: config-2 recipe (N = 10,000); 1, 4: those configs
os.environ["RBG_DEBUG_IMGS"] = str(it)
if cfg == 2:
    N = 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(M, 2, spin=True)
    S = torch.empty((M, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
else:
    Sh, w, _, _ = inputs.make(cfg)
    S = torch.as_tensor(Sh, device="cuda")
ctx = rbg.Context(S, w, 0.0, max(it + 2, 10))
ctx.set_timing(timing)
ctx.step(it + 2)
ctx.sync()
print(f"iteration {it} timing={timing} k={ctx.info()[0]}", flush=True)
ctx.close()
