"""Breakdown of the end-to-end (host S) path on the config-2 workload: H2D bandwidth of a
pinned buffer (one copy vs chunked copies on 2-4 streams) and the phases of rbg_create.

    python scripts/e2e_probe.py [cols]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 409600
N = 10000
dev = torch.device("cuda", 0)
t = inputs.chirp_grid(N)
w = inputs.simpson_weights(N)
q, chi, psi = inputs.chirp_params(M, 2, spin=True)
S = torch.empty((M, N), dtype=torch.complex128, device=dev)
rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
t0 = time.perf_counter()
host = torch.empty(S.shape, dtype=S.dtype, pin_memory=True)
host.copy_(S)
torch.cuda.synchronize()
print(f"pinned alloc + D2H {time.perf_counter() - t0:.2f} s ({S.numel() * 16 / 1e9:.1f} GB)", flush=True)
nbytes = S.numel() * 16


def timed(fn, label):
    torch.cuda.synchronize()
    a = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - a
    print(f"{label:40s} {dt * 1e3:9.1f} ms  {nbytes / dt / 1e9:7.1f} GB/s", flush=True)
    return dt


timed(lambda: S.copy_(host, non_blocking=True), "H2D one copy")
for ns in (2, 4):
    streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    chunks = 64

    def go():
        rows = M // chunks
        for i in range(chunks):
            st = streams[i % ns]
            with torch.cuda.stream(st):
                S[i * rows:(i + 1) * rows].copy_(host[i * rows:(i + 1) * rows], non_blocking=True)
        for st in streams:
            st.synchronize()
    timed(go, f"H2D {chunks} chunks on {ns} streams")
del S
torch.cuda.empty_cache()

Sh = host.numpy()
for rep in range(2):
    torch.cuda.synchronize()
    a = time.perf_counter()
    ctx = rbg.Context(Sh, w, 0.0, 300)
    torch.cuda.synchronize()
    b = time.perf_counter()
    ctx.step(300)
    torch.cuda.synchronize()
    c = time.perf_counter()
    piv, err, Q = ctx.pivots(), ctx.errors(), ctx.basis()
    d = time.perf_counter()
    ctx.close()
    e = time.perf_counter()
    print(f"rep {rep}: create {1e3 * (b - a):.1f} ms ({nbytes / (b - a) / 1e9:.1f} GB/s)  300 it {1e3 * (c - b):.1f} ms"
          f"  outputs {1e3 * (d - c):.1f} ms  close {1e3 * (e - d):.1f} ms  e2e {300 / (d - a):.2f} it/s", flush=True)
