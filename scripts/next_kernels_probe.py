"""Device time (CUDA events on the library stream) of the NEXT-row calls on a config-2 basis:
rbg_eim, rbg_gram, rbg_reconstruct (each includes its own small allocations and copies).

    python scripts/next_kernels_probe.py [cols] [k]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 409600
K = int(sys.argv[2]) if len(sys.argv) > 2 else 300
N = 10000
t = inputs.chirp_grid(N)
w = inputs.simpson_weights(N)
q, chi, psi = inputs.chirp_params(M, 2, spin=True)
S = torch.empty((M, N), dtype=torch.complex128, device="cuda")
rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
st = torch.cuda.Stream()
with rbg.Context(S, w, 0.0, K, stream=st.cuda_stream) as ctx:
    ctx.run()
    for name, fn in [("eim", ctx.eim), ("gram", ctx.gram), ("reconstruct", lambda: ctx.reconstruct(1e-3))]:
        fn()  # warm
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{name:12s} k={K} M={M}: {best:8.2f} ms (best of 3)", flush=True)
