"""CUDA IPC plumbing of the PEER exchange across two processes.

Two processes on cuda:0 (gloo for the handle all-gather) each build a PEER context for their
half of the columns, export their record/send-slot handles, all-gather them and map the
other process's buffers with cudaIpcOpenMemHandle (rbg_peer_connect) -- the path bench.py
takes on a multi-GPU box -- then unmap them on close.  No iteration is run: the ranks'
kernels would wait on each other, which one GPU cannot host (the multi-rank iteration itself
is covered in one process by tests/test_gpu_parity.py with rbg_peer_connect_local).
"""
import pytest

from test_dist_gloo import run_world

pytestmark = pytest.mark.gpu


def _ipc(rank):
    import numpy as np
    import torch

    from paper_1805_06124_b200 import dist as D
    from paper_1805_06124_b200 import inputs, rbg
    torch.cuda.set_device(0)
    S, w, tol, _ = inputs.config1(M=600, N=256)
    off, m = D.partition(600, 2, rank)
    ctx = rbg.Context(S[off:off + m], w, tol, 20, comm=rbg.COMM_PEER, rank=rank, world=2, col_offset=off,
                      M_global=600)
    try:
        mine = ctx.peer_export()
        D.connect_peers(ctx)
        k, _, why = ctx.info()
        return (len(mine), k, why, bool(np.any(np.frombuffer(mine, np.uint8))))
    finally:
        ctx.close()


def test_peer_ipc_handles_map_across_processes():
    res = run_world(_ipc)
    for n, k, why, nonzero in res:
        assert n == 128 and nonzero
        assert k == 0
