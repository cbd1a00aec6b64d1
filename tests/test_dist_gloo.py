"""World-size-2 CPU tests of the multi-GPU host logic over torch.distributed gloo.

* partition / broadcast / max-over-ranks helpers of paper_1805_06124_b200.dist (used by
  bench.py and sharded_context);
* the sharded iteration protocol of DESIGN.md "Multi-GPU", executed with real gloo
  collectives and the CPU oracle's dot / norm / IMGS as each rank's compute: local sweep
  over the rank's column block, local maxloc with the total order, all-gather of one
  {record, candidate column} slot per rank, winner selection, replicated IMGS.  Its result
  must equal the single-process oracle bit for bit, which is the property the CUDA path
  relies on (tests/test_gpu_parity.py::test_sharded_path_on_one_gpu runs the same protocol
  through the library's kernels on one GPU).
"""
from __future__ import annotations

import ctypes
import ctypes.util
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2
_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double] * 3


def _fma(a, b, c):
    return _libm.fma(a, b, c)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        q.put((rank, fn(rank)))
    except Exception as e:  # surface failures to the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_world(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, fn, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(WORLD)]


# ------------------------------------------------------------------------------ helpers

def _helpers(rank):
    from paper_1805_06124_b200 import dist as D
    blocks = [None] * WORLD
    dist.all_gather_object(blocks, D.partition(1001, WORLD, rank))
    payload = bytes(range(128)) if rank == 0 else None
    got = D.broadcast_bytes(payload)
    mx = D.max_over_ranks(1.5 + rank)
    return blocks, got, mx


def test_partition_broadcast_max():
    res = run_world(_helpers)
    for blocks, got, mx in res:
        assert got == bytes(range(128))
        assert mx == 2.5
        offs = sorted(blocks)
        assert offs[0][0] == 0 and sum(b[1] for b in offs) == 1001
        for (o1, n1), (o2, _) in zip(offs, offs[1:]):
            assert o1 + n1 == o2


def test_partition_edge_cases():
    from paper_1805_06124_b200 import dist as D
    for M in (8, 9, 15, 409600 * 8 + 3):
        for P in (1, 2, 3, 8):
            blocks = [D.partition(M, P, r) for r in range(P)]
            assert blocks[0][0] == 0 and sum(b[1] for b in blocks) == M
            assert max(b[1] for b in blocks) - min(b[1] for b in blocks) <= 1
    with pytest.raises(ValueError):
        D.partition(3, 4, 0)


# ------------------------------------------------------------------------------ protocol

def _problem():
    rng = np.random.default_rng(42)
    N, M = 48, 203
    S = rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))
    S[17] = 3.0 * S[150]                               # largest column, duplicated on both
    S[150] = S[17]                                     # ranks: exact tie, lowest index wins
    w = rng.uniform(0.5, 1.5, N)
    return S, w, 0.0, 25


def _sharded_protocol(rank):
    from oracle import oracle as O
    from paper_1805_06124_b200 import dist as D
    S, w, tol, k_max = _problem()
    M, N = S.shape
    L_S, L_I = O.CANONICAL
    off, m_loc = D.partition(M, WORLD, rank)
    Sl = S[off:off + m_loc]
    r2 = np.array([O.nrm(Sl[j], w, L_S) for j in range(m_loc)])
    Q, piv, errs = [], [], []
    stop = None
    for k in range(k_max + 1):
        # local maxloc: value desc, lowest global index on ties
        j = int(np.argmax(r2)) if m_loc else -1
        rec = np.array([r2[j], off + j], dtype=np.float64)
        cand = Sl[j].copy()
        recs = [torch.zeros(2, dtype=torch.float64) for _ in range(WORLD)]
        cols = [torch.zeros(N, dtype=torch.complex128) for _ in range(WORLD)]
        dist.all_gather(recs, torch.from_numpy(rec))
        dist.all_gather(cols, torch.from_numpy(cand))
        best = max(range(WORLD), key=lambda p: (recs[p][0].item(), -recs[p][1].item()))
        m, J = recs[best][0].item(), int(recs[best][1].item())
        err = np.sqrt(max(m, 0.0))
        errs.append(err)
        if m == -np.inf:
            stop = "ALL_SELECTED"
            break
        if err < tol:
            stop = "TOL"
            break
        if k == k_max:
            stop = "KMAX"
            break
        out = O.imgs(np.array(Q).reshape(-1, N), cols[best].numpy(), w, L_I)
        if out is None:
            stop = "RANK"
            break
        q = out[0]
        Q.append(q)
        piv.append(J)
        if off <= J < off + m_loc:
            r2[J - off] = -np.inf
        wq = w * q
        for jj in range(m_loc):
            if r2[jj] != -np.inf:
                c = O.dot(wq, Sl[jj], L_S)
                r2[jj] = r2[jj] - _fma(c.real, c.real, c.imag * c.imag)   # CAC rules 5-6
    return piv, errs, np.array(Q), stop


def test_sharded_protocol_equals_single_process():
    from oracle import oracle as O
    S, w, tol, k_max = _problem()
    ref = O.greedy(S, w, tol, k_max, lanes=O.CANONICAL)
    res = run_world(_sharded_protocol)
    for piv, errs, Q, stop in res:
        assert stop == ref.stop
        assert piv == list(ref.pivots)
        np.testing.assert_array_equal(errs, ref.errors)     # same DAG: bit for bit
        np.testing.assert_array_equal(Q, ref.Q)
    assert ref.pivots[0] == 17 and 150 not in ref.pivots


# ------------------------------------------------------------------------------ sharded Gram

GRAM_M_SPLIT = (0, 8192, 12388)   # rank blocks start at multiples of the 4,096-column chunk


def _gram_problem():
    rng = np.random.default_rng(5)
    k, M = 7, GRAM_M_SPLIT[-1]
    return rng.standard_normal((k, M)) + 1j * rng.standard_normal((k, M))


def _gram_fold_protocol(rank):
    from oracle import oracle as O
    from paper_1805_06124_b200 import dist as D
    R = _gram_problem()
    Rl = R[:, GRAM_M_SPLIT[rank]:GRAM_M_SPLIT[rank + 1]]

    def fold(G):
        # this rank's chunk partials added onto the running sum in chunk order; a one-chunk
        # oracle gram is exactly that chunk's partial (0 + x = x)
        G = G.copy()
        for j0 in range(0, Rl.shape[1], O.GRAM_CHUNK):
            G = G + O.gram(Rl[:, j0:j0 + O.GRAM_CHUNK])
        return G

    return D.fold_over_ranks(fold, R.shape[0])


def test_sharded_gram_fold_equals_single_process():
    """The rank-order Gram fold of dist.sharded_reconstruct over gloo reproduces the oracle's
    single-process chunked Gram bit for bit when the rank blocks are chunk aligned (R33)."""
    from oracle import oracle as O
    ref = O.gram(_gram_problem())
    for G in run_world(_gram_fold_protocol):
        G = G.copy()
        np.fill_diagonal(G, G.diagonal().real)          # the library zeroes it at every fold
        np.testing.assert_array_equal(G, ref)
