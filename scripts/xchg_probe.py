"""Exchange-phase cost C_j per iteration on one GPU: no exchange, NCCL
(one-rank ncclAllGather of the 160 KB slot) and PEER (record stores + wait kernel + NVLink-
capable column read), plus the PEER path with 2/4/8 ranks emulated on one GPU (one stream,
sequential: the C_j there is the wait kernel alone, the sweeps are serialised).

    python scripts/xchg_probe.py [cols] [iters]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 40960
K = int(sys.argv[2]) if len(sys.argv) > 2 else 60
N = 10000
t = inputs.chirp_grid(N)
w = inputs.simpson_weights(N)
q, chi, psi = inputs.chirp_params(M, 2, spin=True)
S = torch.empty((M, N), dtype=torch.complex128, device="cuda")
rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)


def report(name, ctxs, k):
    sw, xc, im = ctxs[0].timings(k)
    piv = ctxs[0].pivots()
    print(f"{name:28s} k={k}  sweep {np.nanmean(sw[3:]) * 1e3:8.1f} us  xchg {np.mean(xc[3:]) * 1e3:7.2f} us"
          f"  imgs {np.mean(im[3:]) * 1e3:7.1f} us  pivots[:4] {piv[:4]}", flush=True)
    return piv


ref = None
for name, comm in [("none", rbg.COMM_NONE), ("nccl world=1", rbg.COMM_NCCL), ("peer world=1", rbg.COMM_PEER)]:
    kw = dict(comm=comm, rank=0, world=1)
    if comm == rbg.COMM_NCCL:
        kw["nccl_id"] = rbg.unique_id()
    with rbg.Context(S, w, 0.0, K, **kw) as ctx:
        ctx.set_timing(True)
        ctx.run()
        piv = report(name, [ctx], ctx.info()[0])
        assert ref is None or np.array_equal(piv, ref)
        ref = piv

for world in (2, 4, 8):
    stream = torch.cuda.Stream()
    b = [M * p // world for p in range(world + 1)]
    ctxs = [rbg.Context(S[b[p]:b[p + 1]], w, 0.0, K, stream=stream.cuda_stream, comm=rbg.COMM_PEER, rank=p,
                        world=world, col_offset=b[p], M_global=M) for p in range(world)]
    rbg.peer_connect_local(ctxs)
    for c in ctxs:
        c.set_timing(True)
    for _ in range(K + 1):
        for c in ctxs:
            c.iter_local()
        for c in ctxs:
            c.iter_finish()
    piv = report(f"peer {world} ranks emulated", ctxs, ctxs[0].info()[0])
    assert np.array_equal(piv, ref)
    for c in ctxs:
        c.close()
