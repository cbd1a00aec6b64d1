"""Seeded synthetic inputs for the five BASELINE.json configs (host, numpy).

This module holds only the input recipe: no arithmetic of the
method.  Both the CUDA path and the CPU oracle consume the bytes it returns.

Every generator returns ``(S, w, tol, k_max)`` with ``S`` an (M, N) C-order array,
i.e. column-major N x M with snapshot j in row ``S[j]`` (SPEC.md:79 disk convention),
and ``w`` the (N,) quadrature weights of the inner product <x, y>_w.

The paper's own snapshots are IMRPhenomPv2 gravitational waveforms from LALSuite
(PAPER.md:820-834), which are not available here; the chirp family below stands in for
them with the paper's shapes (N = 10,000 rows, M = 100 columns per core,
PAPER.md:1096-1108), as BASELINE.json prescribes.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 1805061240  # numpy default_rng(SEED_BASE + config index)
CHIRP_F0 = 4.0          # DESIGN.md reading R19 (f0 unspecified in BASELINE.json)
CHIRP_EPS = 1e-3        # BASELINE.json config 1


def rng_for(cfg: int) -> np.random.Generator:
    return np.random.default_rng(SEED_BASE + cfg)


def simpson_weights(N: int) -> np.ndarray:
    """Composite Simpson (h/3)(1,4,2,...,4,1) on points 0..N-2 plus a trapezoid on the
    last interval, h = 1/N (reading R20).  N must be even and >= 4."""
    if N < 4 or N % 2:
        raise ValueError("simpson_weights needs even N >= 4")
    h = 1.0 / N
    w = np.zeros(N)
    npts = N - 1                       # points 0..N-2, an odd count -> even intervals
    w[:npts] = 2.0
    w[1:npts - 1:2] = 4.0
    w[0] = 1.0
    w[npts - 1] = 1.0
    w[:npts] *= h / 3.0
    w[N - 2] += h / 2.0
    w[N - 1] += h / 2.0
    return w


def chirp_grid(N: int) -> np.ndarray:
    """t_i = -1 + i/N, i = 0..N-1 (t in [-1, 0), reading R20)."""
    return -1.0 + np.arange(N) / N


def chirp_params(M: int, cfg: int, spin: bool):
    """Per-column parameters, drawn in a fixed order: q (log-uniform [1,10]),
    chi (U[-1,1], spin configs only), psi (U[0, 2 pi))."""
    rng = rng_for(cfg)
    q = 10.0 ** rng.uniform(0.0, 1.0, M)
    chi = rng.uniform(-1.0, 1.0, M) if spin else np.zeros(M)
    psi = rng.uniform(0.0, 2.0 * np.pi, M)
    return q, chi, psi


def chirp_columns(t: np.ndarray, w: np.ndarray, q, chi, psi, spin: bool) -> np.ndarray:
    """h_j(t) = A(t) (1 + 0.3 chi_j cos 3 phi) exp(i (phi + psi_j)), normalised to
    ||h_j||_w = 1 (readings R21, R22).  Returns (len(q), N) complex128."""
    x = (-t + CHIRP_EPS)
    A = x ** -0.25
    base = -2.0 * np.pi * CHIRP_F0 * x ** 0.625 / 0.625   # phi = q_j * base(t)
    phi = np.asarray(q)[:, None] * base[None, :]
    amp = A[None, :] * (1.0 + 0.3 * np.asarray(chi)[:, None] * np.cos(3.0 * phi)) if spin \
        else np.broadcast_to(A[None, :], phi.shape)
    H = amp * np.exp(1j * (phi + np.asarray(psi)[:, None]))
    norms = np.sqrt((np.abs(H) ** 2) @ w)
    return np.ascontiguousarray(H / norms[:, None])


_host_lib = None
HOST_SRC = __file__.rsplit("/", 1)[0] + "/inputs_host.c"
HOST_LIB = __file__.rsplit("/", 1)[0] + "/libinputs_host.so"


def build_host(force: bool = False) -> str:
    """Compile the OpenMP host generator (inputs_host.c: the recipe only)."""
    import os
    import subprocess
    if not force and os.path.exists(HOST_LIB) and os.path.getmtime(HOST_LIB) >= os.path.getmtime(HOST_SRC):
        return HOST_LIB
    tmp = HOST_LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", HOST_SRC, "-o", tmp, "-lm"])
    os.replace(tmp, HOST_LIB)
    return HOST_LIB


def chirp_columns_host(t: np.ndarray, w: np.ndarray, q, chi, psi, spin: bool, out=None, threads: int = 0) -> np.ndarray:
    """chirp_columns with every host core (inputs_host.c, OpenMP over columns): the full
    409,600-column matrix in seconds instead of minutes.  Equal to chirp_columns to rounding
    (another libm); used where only the workload's shape and values matter (the reference
    arm's timing), never for a bit-exact comparison."""
    import ctypes
    global _host_lib
    if _host_lib is None:
        _host_lib = ctypes.CDLL(build_host())
        dp = ctypes.POINTER(ctypes.c_double)
        _host_lib.rbg_inputs_chirp.argtypes = [dp, ctypes.c_int64, ctypes.c_int64, dp, dp, dp, dp, dp, dp,
                                               ctypes.c_int, ctypes.c_int]
        _host_lib.rbg_inputs_chirp.restype = None
    x = (-np.asarray(t, dtype=np.float64) + CHIRP_EPS)
    A = np.ascontiguousarray(x ** -0.25)
    base = np.ascontiguousarray(-2.0 * np.pi * CHIRP_F0 * x ** 0.625 / 0.625)
    wv = np.ascontiguousarray(w, dtype=np.float64)
    qv, cv, pv = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, chi, psi))
    M, N = len(qv), len(A)
    if out is None:
        out = np.empty((M, N), np.complex128)
    assert out.shape == (M, N) and out.dtype == np.complex128 and out.flags.c_contiguous

    def p(a):
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    if threads <= 0:
        import os
        threads = len(os.sched_getaffinity(0))        # every core (torchrun workers default to 1)
    _host_lib.rbg_inputs_chirp(p(out.view(np.float64)), N, M, p(A), p(base), p(wv), p(qv), p(cv), p(pv),
                               1 if spin else 0, threads)
    return out


def config0(M: int = 512, N: int = 256):
    """Runge family: s_j(x_i) = 1/(1 + 25 (x_i - mu_j)^2), x uniform on [-1, 1] with
    endpoints (reading R23), mu_j ~ U[-1, 1]; w_i = 2/256; tol 1e-10, k_max 128."""
    rng = rng_for(0)
    mu = rng.uniform(-1.0, 1.0, M)
    x = -1.0 + 2.0 * np.arange(N) / (N - 1)
    S = 1.0 / (1.0 + 25.0 * (x[None, :] - mu[:, None]) ** 2)
    w = np.full(N, 2.0 / 256.0)
    return np.ascontiguousarray(S), w, 1e-10, min(128, N, M)


def config1(M: int = 20000, N: int = 2000):
    """Complex chirps, 2,000 x 20,000, Simpson weights; tol 1e-12, k_max 400."""
    t = chirp_grid(N)
    w = simpson_weights(N)
    q, chi, psi = chirp_params(M, 1, spin=False)
    return chirp_columns(t, w, q, chi, psi, spin=False), w, 1e-12, min(400, N, M)


def config2(M: int = 409600, N: int = 10000, cfg: int = 2):
    """Spin-modulated complex chirps 10,000 x 409,600 (~65.5 GB); tol 0 (R24), k_max 300.
    Full size is only generated on the device (bench); host use is for reduced M."""
    t = chirp_grid(N)
    w = simpson_weights(N)
    q, chi, psi = chirp_params(M, cfg, spin=True)
    return chirp_columns(t, w, q, chi, psi, spin=True), w, 0.0, min(300, N, M)


def config4(M: int = 65536, N: int = 4096, r: int = 512):
    """S = U diag(sigma) V^T with Haar U (N x r), V (M x r), sigma_i = 10^(-i/25),
    w_i ~ U[0.5, 1.5]; tol 1e-13, k_max 512 (reading R24)."""
    rng = rng_for(4)

    def haar(n, k):
        G = rng.standard_normal((n, k))
        Qm, Rm = np.linalg.qr(G)
        return Qm * np.sign(np.diag(Rm))[None, :]

    U = haar(N, r)
    V = haar(M, r)
    w = rng.uniform(0.5, 1.5, N)
    sigma = 10.0 ** (-np.arange(r) / 25.0)
    S_T = (V * sigma[None, :]) @ U.T          # (M, N) = (U diag(sigma) V^T)^T
    return np.ascontiguousarray(S_T), w, 1e-13, min(r, N, M), (U, sigma, V)


def make(cfg: int, **kw):
    """Config by index; keyword overrides (M=..., N=...) give reduced-size variants."""
    if cfg == 0:
        return config0(**kw)
    if cfg == 1:
        return config1(**kw)
    if cfg in (2, 3):
        return config2(cfg=cfg, **kw)
    if cfg == 4:
        return config4(**kw)[:4]
    raise ValueError(cfg)
