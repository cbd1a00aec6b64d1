"""ctypes front end of the CPU oracle (oracle/rbg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs, never by the product package
``paper_1805_06124_b200``.  It shares no code with the CUDA path.

Functions follow arXiv 1805.06124 (PAPER.md line numbers):
  * ``greedy``  -- Algorithm 3 RB-greedy with the residual recurrence (PAPER.md:452-477,
    846-866) and Hoffmann IMGS;
  * ``imgs``    -- the IMGS step alone;
  * ``dot`` / ``nrm`` -- the weighted inner product and norm in the canonical order.

Parity unpinned: the exact pivot sequence below the recurrence floor (R8) and the
exact k of a RANK stop are fixed only by the canonical summation order, not by the paper.

Lane counts: ``L_S`` (sweep) and ``L_I`` (IMGS).  ``L_S = L_I = 1`` is the plain
sequential-sum mode; ``CANONICAL = (32, 2048)`` is the order of DESIGN.md's
canonical arithmetic contract.  These numbers are written here from DESIGN.md, not
read from the CUDA library.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rbg_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

CANONICAL = (32, 2048)  # (L_S, L_I): DESIGN.md "Canonical arithmetic contract"
CANONICAL_CGS = (32, 256)  # (L_S, L_C) for the CGSCI variant (CAC rule 11)
PLAIN = (1, 1)

STOP_NAMES = {0: "NONE", 1: "TOL", 2: "KMAX", 3: "RANK", 4: "ALL_SELECTED"}


def _cpu_has_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " fma" in f.read()
    except OSError:
        return False


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-ffp-contract=off: no implicit fma)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    flags = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]
    if _cpu_has_fma():
        flags.append("-mfma")
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *flags, SRC, "-o", tmp, "-lm"])
    os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.orc_dot.argtypes = [d, d, i64, ctypes.c_int, ctypes.c_int, d, d]
        L.orc_dot.restype = None
        L.orc_nrm.argtypes = [d, d, i64, ctypes.c_int, ctypes.c_int]
        L.orc_nrm.restype = ctypes.c_double
        L.orc_imgs.argtypes = [d, d, i64, i64, d, d, i64, ctypes.c_int, ctypes.c_int,
                               d, d, d, d, ctypes.POINTER(ctypes.c_int)]
        L.orc_imgs.restype = ctypes.c_int
        L.orc_greedy.argtypes = [d, i64, i64, i64, d, ctypes.c_int, ctypes.c_double, i64,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, i64, i64, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(i64), d, d, d, d,
                                 ctypes.POINTER(ctypes.c_int), d, d,
                                 ctypes.POINTER(ctypes.c_int), d, d, d]
        L.orc_greedy.restype = i64
        L.orc_validate.argtypes = [d, i64, i64, d, i64, i64, d, i64, ctypes.c_int, ctypes.c_int,
                                   d, d, ctypes.c_int]
        L.orc_validate.restype = None
        L.orc_gram.argtypes = [d, i64, i64, ctypes.c_int, i64, d]
        L.orc_gram.restype = None
        L.orc_eim.argtypes = [d, i64, i64, ctypes.POINTER(i64), d]
        L.orc_eim.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _flat(x: np.ndarray) -> tuple[np.ndarray, int]:
    """Return (float64 view, cplx flag) of a contiguous real or complex array."""
    x = np.ascontiguousarray(x)
    if np.iscomplexobj(x):
        return x.astype(np.complex128, copy=False).view(np.float64), 1
    return x.astype(np.float64, copy=False), 0


def dot(xt: np.ndarray, y: np.ndarray, L: int = 1) -> complex:
    """sum_i conj(xt_i) y_i in the CAC order with L lanes (DESIGN.md rule 2-3)."""
    xf, c1 = _flat(xt)
    yf, c2 = _flat(y)
    assert c1 == c2 and xt.shape == y.shape
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().orc_dot(_p(xf), _p(yf), xt.size, c1, L, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value) if c1 else re.value


def nrm(y: np.ndarray, w: np.ndarray, L: int = 1) -> float:
    """sum_i w_i |y_i|^2 in the CAC order (DESIGN.md rule 4)."""
    yf, c = _flat(y)
    w = np.ascontiguousarray(w, dtype=np.float64)
    return lib().orc_nrm(_p(yf), _p(w), y.size, c, L)


def imgs(Q: np.ndarray, v: np.ndarray, w: np.ndarray, L: int = 1):
    """Hoffmann IMGS of v against the k columns of Q (Q given as (k, N) rows = columns).

    Returns (q, coeff, n, nu) or None when the candidate is degenerate (stop RANK).
    """
    w = np.ascontiguousarray(w, dtype=np.float64)
    cplx = np.iscomplexobj(Q) or np.iscomplexobj(v)
    dt = np.complex128 if cplx else np.float64
    Q = np.ascontiguousarray(Q, dtype=dt).reshape(-1, v.shape[0])
    k, N = Q.shape
    WQ = np.ascontiguousarray(Q * w[None, :])
    vv = np.array(v, dtype=dt, copy=True)
    q = np.zeros(N, dt)
    wq = np.zeros(N, dt)
    coeff = np.zeros(max(k, 1), dt)
    n = ctypes.c_double()
    nu = ctypes.c_int()
    Qf = Q.view(np.float64) if k else np.zeros(1)
    WQf = WQ.view(np.float64) if k else np.zeros(1)
    ok = lib().orc_imgs(_p(Qf), _p(WQf), N * (2 if cplx else 1), k, _p(vv.view(np.float64)),
                        _p(w), N, int(cplx), L, _p(q.view(np.float64)), _p(wq.view(np.float64)),
                        _p(coeff.view(np.float64)), ctypes.byref(n), ctypes.byref(nu))
    if not ok:
        return None
    return q, coeff[:k], n.value, nu.value


@dataclass
class GreedyResult:
    k: int
    stop: str
    pivots: np.ndarray    # (k,) int64 global column ids
    Q: np.ndarray         # (k, N): row i is basis vector q_i  (column-major N x k)
    R: np.ndarray         # (k, M): R[i, j] = <q_i, s_j>_w from the sweep
    errors: np.ndarray    # (k+1,) err_0 .. err_k
    nu: np.ndarray        # (k,) IMGS sweeps
    rdiag: np.ndarray     # (k,) IMGS norms (R(k,k) of the new column)
    r2: np.ndarray        # (M,) final squared residuals (selected = -inf)
    t_sweep: np.ndarray   # (k,) seconds per sweep
    t_imgs: np.ndarray    # (k,) seconds per IMGS
    t_iter: np.ndarray    # (k,) seconds per whole iteration (argmax + IMGS + sweep)


def greedy(S: np.ndarray, w: np.ndarray, tol: float, k_max: int,
           lanes: tuple[int, int] = CANONICAL, threads: int = 0,
           max_iters: int = -1, resume: "GreedyResult | None" = None,
           ortho: str = "mgs", residual: str = "recurrence") -> GreedyResult:
    """RB-greedy (Algorithm 3) on S given as an (M, N) C-order array (column-major N x M).

    ``lanes=(L_S, L_I)``; ``threads=0`` lets OpenMP choose.  ``resume`` continues from a
    previous state whose R / r2 already cover all M columns (enrichment).  ``ortho="cgs"``
    uses Hoffmann's iterated classical GS (pass lanes=CANONICAL_CGS for GPU parity).
    ``residual="explicit"`` keeps Algorithm 2's explicitly updated columns (CAC rule 12).
    """
    Sf, cplx = _flat(S)
    M, N = S.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    assert w.shape == (N,)
    nv = 2 if cplx else 1
    dt = np.complex128 if cplx else np.float64
    piv = np.zeros(k_max, np.int64)
    Q = np.zeros((k_max, N), dt)
    WQ = np.zeros((k_max, N), dt)
    R = np.zeros((k_max, M), dt)
    err = np.zeros(k_max + 1)
    nu = np.zeros(k_max, np.int32)
    rdiag = np.zeros(k_max)
    r2 = np.zeros(M)
    k0 = -1
    if resume is not None:
        assert residual == "recurrence"
        k0 = resume.k
        assert resume.R.shape == (k0, M) and resume.r2.shape == (M,)
        piv[:k0] = resume.pivots
        Q[:k0] = resume.Q
        WQ[:k0] = resume.Q * w[None, :]
        R[:k0] = resume.R
        err[:k0 + 1] = resume.errors[:k0 + 1]
        nu[:k0] = resume.nu
        rdiag[:k0] = resume.rdiag
        r2[:] = resume.r2
    stop = ctypes.c_int()
    ts = np.zeros(k_max)
    ti = np.zeros(k_max)
    tt = np.zeros(k_max)
    k = lib().orc_greedy(
        _p(Sf), N, M, N * nv, _p(w), cplx, float(tol), int(k_max), lanes[0], lanes[1],
        threads, int(max_iters), int(k0), 1 if ortho == "cgs" else 0, 1 if residual == "explicit" else 0,
        piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _p(Q.view(np.float64)),
        _p(WQ.view(np.float64)), _p(R.view(np.float64)), _p(err),
        nu.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _p(rdiag), _p(r2),
        ctypes.byref(stop), _p(ts), _p(ti), _p(tt))
    if k < 0:
        raise ValueError("oracle: bad arguments")
    return GreedyResult(k=int(k), stop=STOP_NAMES[stop.value], pivots=piv[:k].copy(),
                        Q=Q[:k].copy(), R=R[:k].copy(), errors=err[:k + 1].copy(),
                        nu=nu[:k].copy(), rdiag=rdiag[:k].copy(), r2=r2, t_sweep=ts[:k].copy(),
                        t_imgs=ti[:k].copy(), t_iter=tt[:k].copy())


def validate(Q: np.ndarray, V: np.ndarray, w: np.ndarray, L_S: int = CANONICAL[0], threads: int = 0):
    """Out-of-sample validation against the basis Q (k, N): returns (err, C, e2) with
    C (k, M_v) the coefficients <q_i, v_j>_w and e2 the recurrence residual (DESIGN.md f-1)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    cplx = np.iscomplexobj(Q) or np.iscomplexobj(V)
    dt = np.complex128 if cplx else np.float64
    V = np.ascontiguousarray(V, dtype=dt)
    M_v, N = V.shape
    k = Q.shape[0]
    WQ = np.ascontiguousarray(np.asarray(Q, dtype=dt) * w[None, :]) if k else np.zeros((1, N), dt)
    C = np.zeros((max(k, 1), M_v), dt)
    e2 = np.zeros(M_v)
    nv = 2 if cplx else 1
    lib().orc_validate(_p(WQ.view(np.float64)), N * nv, k, _p(V.view(np.float64)), M_v, N * nv, _p(w), N,
                       int(cplx), L_S, _p(C.view(np.float64)), _p(e2), threads)
    return np.sqrt(np.maximum(e2, 0.0)), C[:k], e2


def enrich(S: np.ndarray, V: np.ndarray, w: np.ndarray, tol: float, k_max: int, rounds: int = 3,
           lanes: tuple[int, int] = CANONICAL):
    """Iterative refinement (SPEC enrich): greedy on S; per round validate V,
    append every failing column (err >= tol) not appended before to the training set and
    continue the greedy from its state.  Returns (result, S_final, history, passed)."""
    res = greedy(S, w, tol, k_max, lanes=lanes)
    added = np.zeros(V.shape[0], bool)
    history = []
    for _ in range(rounds):
        err, _, _ = validate(res.Q, V, w, lanes[0])
        history.append(float(err.max()) if err.size else 0.0)
        fail = (err >= tol) & ~added
        if not fail.any():
            return res, S, history, bool(np.all(err < tol))
        F = V[fail]
        added |= fail
        _, C, e2 = validate(res.Q, F, w, lanes[0])
        S = np.concatenate([S, F])
        res.R = np.concatenate([res.R, C], axis=1)
        res.r2 = np.concatenate([res.r2, e2])
        res = greedy(S, w, tol, k_max, lanes=lanes, resume=res)
    err, _, _ = validate(res.Q, V, w, lanes[0])
    history.append(float(err.max()) if err.size else 0.0)
    return res, S, history, bool(np.all(err < tol))


GRAM_CHUNK = 4096  # DESIGN.md reading R30 (written here from the document, not the library)


def gram(R: np.ndarray, chunk: int = GRAM_CHUNK) -> np.ndarray:
    """G = R R^H (k x k, complex) in the chunked order of DESIGN.md R30."""
    Rf, cplx = _flat(R)
    k, M = R.shape
    buf = np.zeros(k * k, np.complex128)            # column-major k x k
    if k:
        lib().orc_gram(_p(Rf), k, M, cplx, chunk, _p(buf.view(np.float64)))
    return buf.reshape((k, k), order="F")


def reconstruct(res: GreedyResult, tau2: float = 0.0, kr_max: int = 0):
    """Algorithm 4: SVD of R(1:k, :) through its Gram matrix (LAPACK
    eigh as the library step), sigma descending (ties by index), kr = #{sigma > tau2} (prefix,
    capped at kr_max), X = Q V(:, 1:kr).  Returns (sigma, kr, X (kr, N), V)."""
    k = res.k
    if k == 0:
        return np.zeros(0), 0, np.zeros((0, res.Q.shape[1] if res.Q.ndim == 2 else 0)), None
    G = gram(res.R)
    lam, V = np.linalg.eigh(G)
    order = sorted(range(k), key=lambda i: (-lam[i], i))
    sigma = np.sqrt(np.maximum(lam[order], 0.0))
    kr = 0
    while kr < k and sigma[kr] > tau2:
        kr += 1
    if kr_max:
        kr = min(kr, kr_max)
    Vs = V[:, order]
    X = (res.Q.T @ Vs[:, :kr]).T
    return sigma, kr, X, Vs


def eim(Q: np.ndarray):
    """Greedy EIM nodes of the basis Q (k, N) (R31): (nodes (k,), B = Q(nodes, :)
    as a (k, k) matrix with B[a, b] = q_b(nodes[a])), or None if degenerate."""
    k, N = Q.shape
    Qc = np.ascontiguousarray(Q, dtype=np.complex128)
    nodes = np.zeros(max(k, 1), np.int64)
    buf = np.zeros(max(k, 1) ** 2, np.complex128)
    if k == 0:
        return nodes[:0], np.zeros((0, 0))
    ok = lib().orc_eim(_p(Qc.view(np.float64)), k, N, nodes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                       _p(buf.view(np.float64)))
    if not ok:
        return None
    B = buf.reshape((k, k), order="F")
    return nodes, (B if np.iscomplexobj(Q) else B.real.copy())
