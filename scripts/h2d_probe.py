"""H2D bandwidth from pinned host memory on this box: one copy vs the same bytes as chunks over
1, 2 or 4 streams (copy engines), and one copy followed by a device-side scan vs chunks with the
scan of chunk i overlapping the copy of chunk i+1 (torch only; what rbg_create's upload could use)."""
import json
import time

import torch

GB = 1 << 30
n = 8 * GB
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()


def timed(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


out = {}
out["one_copy_GBps"] = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = 256 * 1024 * 1024

    def run():
        for i, off in enumerate(range(0, n, chunk)):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        for s in streams:
            s.synchronize()
    out[f"chunks256M_{ns}streams_GBps"] = n / timed(run) / 1e9
print(json.dumps(out))
