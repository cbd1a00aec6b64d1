"""rbg_create from pinned host memory: wall time of the create (upload + finiteness scan +
allocations) for a complex 10,000 x M snapshot block (default 102,400 columns = 16.4 GB)."""
import json
import sys
import time
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import rbg  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 102400
N = 10000
h = torch.empty((M, N), dtype=torch.complex128, pin_memory=True)
h.real.fill_(1.0)
h.imag.fill_(0.5)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = rbg.Context(h, None, 0.0, 300)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    ctx.close()
print(json.dumps({"cols": M, "GB": M * N * 16 / 1e9, "create_s": ts, "GBps_best": M * N * 16 / 1e9 / min(ts)}))
