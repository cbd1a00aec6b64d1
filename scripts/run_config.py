#!/usr/bin/env python
"""Run one BASELINE config's whole greedy through rbg_run (for ncu launch lists):
    python scripts/run_config.py <0|1|4> [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
S, w, tol, k_max = inputs.make(cfg)
St = torch.as_tensor(S, device="cuda")
for _ in range(reps):
    with rbg.Context(St, w, tol, k_max) as ctx:
        ctx.run()
        print(cfg, ctx.info(), flush=True)
