"""Small runs of every kernel family for compute-sanitizer (one tool per invocation)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

S, w, tol, k_max = inputs.config1(M=700, N=300)
for kw in ({}, {"ortho": "cgs"}, {"residual": "explicit"}):
    with rbg.Context(S, w, tol, 40, **kw) as ctx:
        ctx.run()
        ctx.result()
        if not kw:
            ctx.validate(S[:50])
            ctx.gram()
            ctx.reconstruct(1e-3)
            ctx.eim()
            ctx.add_columns(S[:20] * 1.5)
            ctx.run()
Sr = np.random.default_rng(1).standard_normal((100, 257))
rbg.greedy(Sr, None, 0.0, 30)
ctxs = [rbg.Context(S[p * 350:(p + 1) * 350], w, tol, 20, comm=rbg.COMM_EXTERNAL, rank=p, world=2,
                    col_offset=p * 350, M_global=700) for p in range(2)]
for _ in range(21):
    for c in ctxs:
        c.iter_local()
    rbg.emulate_allgather(ctxs)
    for c in ctxs:
        c.iter_finish()
print("ok", [c.info() for c in ctxs])
import torch  # noqa: E402

st = torch.cuda.Stream()
pctx = [rbg.Context(S[p * 350:(p + 1) * 350], w, tol, 20, stream=st.cuda_stream, comm=rbg.COMM_PEER, rank=p,
                    world=2, col_offset=p * 350, M_global=700) for p in range(2)]
rbg.peer_connect_local(pctx)
for _ in range(21):
    for c in pctx:
        c.iter_local()
    for c in pctx:
        c.iter_finish()
print("peer ok", [c.info() for c in pctx])
