"""Python binding of librbg.so (include/rbg.h): argument marshalling only.

Every step of the RB-greedy hot path runs in the library's CUDA kernels; this module only
turns numpy arrays / torch tensors into pointers and back.  There is no CPU fallback:
if the extension is missing or no GPU is present, calls raise.

    res = greedy(S, w, tol, k_max)      # S: (M, N) host numpy or cuda torch tensor

``S`` is given as (M, N) C-order (snapshot j = S[j]), which is the column-major N x M
matrix of the paper.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "librbg.so")

OK, EINVAL, ENONFINITE, ENOMEM, ECUDA, ENCCL, ESTATE = range(7)
STATUS = {0: "OK", 1: "EINVAL", 2: "ENONFINITE", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ESTATE"}
STOP = {0: "NONE", 1: "TOL", 2: "KMAX", 3: "RANK", 4: "ALL_SELECTED", 5: "PEER_TIMEOUT"}
REAL_F64, COMPLEX_F64 = 1, 2
MEM_HOST, MEM_DEVICE = 0, 1
COMM_NONE, COMM_NCCL, COMM_EXTERNAL, COMM_PEER = 0, 1, 2, 3
PEER_HANDLE_BYTES = 128
ORTHO = {"mgs": 0, "cgs": 1}
RESIDUAL = {"recurrence": 0, "explicit": 1}


class RbgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Desc(ctypes.Structure):
    _fields_ = [
        ("S", ctypes.c_void_p), ("S_mem", ctypes.c_int), ("N", ctypes.c_int64),
        ("M", ctypes.c_int64), ("ld", ctypes.c_int64), ("borrow", ctypes.c_int),
        ("w", ctypes.c_void_p), ("w_mem", ctypes.c_int), ("dtype", ctypes.c_int),
        ("tol", ctypes.c_double), ("k_max", ctypes.c_int64), ("stream", ctypes.c_void_p),
        ("device", ctypes.c_int), ("check_finite", ctypes.c_int), ("comm", ctypes.c_int),
        ("rank", ctypes.c_int), ("world", ctypes.c_int), ("col_offset", ctypes.c_int64),
        ("M_global", ctypes.c_int64), ("nccl_id", ctypes.c_uint8 * 128), ("ortho", ctypes.c_int),
        ("residual", ctypes.c_int), ("peer_timeout_ms", ctypes.c_int64),
    ]


class Stats(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("sweeps", ctypes.c_int64), ("t_init_ms", ctypes.c_double),
                ("t_sweep_ms", ctypes.c_double), ("t_xchg_ms", ctypes.c_double),
                ("t_imgs_ms", ctypes.c_double), ("t_total_ms", ctypes.c_double),
                ("t_gap_ms", ctypes.c_double), ("noop_iters", ctypes.c_int64)]


# (name, argtypes, restype) for every symbol include/rbg.h and include/rbg_gen.h declare
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
SYMBOLS = {
    "rbg_desc_init": ([ctypes.POINTER(Desc)], None),
    "rbg_create": ([ctypes.POINTER(_P), _P, _I64, _I64, _P, ctypes.c_double, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_create_ex": ([ctypes.POINTER(_P), ctypes.POINTER(Desc)], ctypes.c_int),
    "rbg_get_unique_id": ([ctypes.POINTER(ctypes.c_uint8)], ctypes.c_int),
    "rbg_run": ([_P], ctypes.c_int),
    "rbg_step": ([_P, _I64], ctypes.c_int),
    "rbg_set_timing": ([_P, ctypes.c_int], ctypes.c_int),
    "rbg_set_graph_batch": ([_P, ctypes.c_int], ctypes.c_int),
    "rbg_sync": ([_P], ctypes.c_int),
    "rbg_result_info": ([_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "rbg_get_pivots": ([_P, _P], ctypes.c_int),
    "rbg_get_errors": ([_P, _P], ctypes.c_int),
    "rbg_get_nu": ([_P, _P], ctypes.c_int),
    "rbg_get_rdiag": ([_P, _P], ctypes.c_int),
    "rbg_get_basis": ([_P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_get_R": ([_P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_get_r2": ([_P, _P, ctypes.c_int], ctypes.c_int),
    "rbg_get_stats": ([_P, ctypes.POINTER(Stats)], ctypes.c_int),
    "rbg_get_timings": ([_P, _P, _P, _P, _I64], ctypes.c_int),
    "rbg_iter_local": ([_P], ctypes.c_int),
    "rbg_iter_finish": ([_P], ctypes.c_int),
    "rbg_xchg_buffers": ([_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "rbg_emulate_allgather": ([ctypes.POINTER(_P), ctypes.c_int], ctypes.c_int),
    "rbg_peer_export": ([_P, ctypes.POINTER(ctypes.c_uint8)], ctypes.c_int),
    "rbg_peer_connect": ([_P, ctypes.POINTER(ctypes.c_uint8)], ctypes.c_int),
    "rbg_peer_connect_local": ([ctypes.POINTER(_P), ctypes.c_int], ctypes.c_int),
    "rbg_lanes": ([ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], None),
    "rbg_debug_set_canary": ([ctypes.c_int], None),
    "rbg_debug_canary_violations": ([], ctypes.c_int64),
    "rbg_version": ([], ctypes.c_char_p),
    "rbg_last_error": ([], ctypes.c_char_p),
    "rbg_destroy": ([_P], None),
    "rbg_validate": ([_P, _P, _I64, _I64, ctypes.c_int, _P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_add_columns": ([_P, _P, _I64, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_add_columns_ex": ([_P, _P, _I64, _I64, ctypes.c_int, _I64, _I64], ctypes.c_int),
    "rbg_gram": ([_P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_restore": ([_P, _I64, _P, _P, _P, _P, _P, _I64, _P, _I64, _P, ctypes.c_int], ctypes.c_int),
    "rbg_reconstruct": ([_P, ctypes.c_double, _I64, ctypes.POINTER(_I64), _P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_eim": ([_P, _P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_gram_fold": ([_P, _P, _I64, ctypes.c_int], ctypes.c_int),
    "rbg_reconstruct_gram": ([_P, _P, _I64, ctypes.c_int, ctypes.c_double, _I64, ctypes.POINTER(_I64), _P, _P, _I64,
                              ctypes.c_int], ctypes.c_int),
    "rbg_gen_chirp": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P], ctypes.c_int),
}

_lib = None


def lib():
    """Load librbg.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1805_06124_b200.build` "
                              "or __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (argt, rest) in SYMBOLS.items():
            f = getattr(L, name)
            f.argtypes = argt
            f.restype = rest
        _lib = L
    return _lib


def _host_out(shape, dtype) -> np.ndarray:
    """Output array for a device-to-host copy: from 1 MB to 256 MB it is page-locked (torch's
    caching host allocator, reused across calls), so the copy runs at link speed instead of
    through the driver's pageable staging (48 MB of X: 11.9 ms pageable); larger outputs (R of a
    big context) stay pageable rather than pin gigabytes of host memory."""
    dtype = np.dtype(dtype)
    if (1 << 20) <= int(np.prod(shape)) * dtype.itemsize <= (256 << 20):
        import torch
        tdt = torch.complex128 if dtype == np.complex128 else torch.float64
        return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()
    return np.zeros(shape, dtype)


def _check(status: int):
    if status != OK:
        raise RbgError(status, lib().rbg_last_error().decode())


def set_canary(on: bool):
    """Canary tails on every device buffer allocated from now on (rbg_debug_set_canary)."""
    lib().rbg_debug_set_canary(1 if on else 0)


def canary_violations() -> tuple[int, str]:
    """(violations so far, first message) after checking every live canaried buffer."""
    n = int(lib().rbg_debug_canary_violations())
    return n, (lib().rbg_last_error().decode() if n else "")


def lanes() -> tuple[int, int]:
    a, b = ctypes.c_int(), ctypes.c_int()
    lib().rbg_lanes(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def version() -> str:
    return lib().rbg_version().decode()


def unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().rbg_get_unique_id(buf))
    return bytes(buf)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class Result:
    k: int
    stop: str
    pivots: np.ndarray   # (k,) global column ids
    errors: np.ndarray   # (k+1,)
    nu: np.ndarray       # (k,)
    rdiag: np.ndarray    # (k,)
    Q: np.ndarray | None   # (k, N)
    R: np.ndarray | None   # (k, M_loc)
    r2: np.ndarray | None  # (M_loc,)


class Context:
    """One rbg_ctx.  ``S`` is an (M_loc, N) array: host numpy (copied) or a CUDA torch
    tensor (borrowed when contiguous, i.e. ld = N)."""

    def __init__(self, S, w=None, tol: float = 0.0, k_max: int = 1, *, stream=None,
                 comm: int = COMM_NONE, rank: int = 0, world: int = 1, col_offset: int = 0,
                 M_global: int = 0, nccl_id: bytes | None = None, check_finite: bool = True,
                 borrow: bool = True, ortho: str = "mgs", residual: str = "recurrence",
                 peer_timeout_ms: int = 0):
        L = lib()
        d = Desc()
        L.rbg_desc_init(ctypes.byref(d))
        self._keep = []
        if _is_torch(S):
            import torch
            if not S.is_cuda:
                S = S.numpy()
            else:
                if S.dim() != 2:
                    raise ValueError("S must be 2-D (M, N)")
                cplx = S.is_complex()
                if S.dtype not in (torch.float64, torch.complex128):
                    raise ValueError("S must be float64 or complex128")
                if S.stride(1) != 1:
                    raise ValueError("S rows (snapshots) must be contiguous")
                d.S = S.data_ptr()
                d.S_mem = MEM_DEVICE
                d.ld = S.stride(0)
                d.borrow = 1 if borrow else 0
                d.M, d.N = S.shape
                d.dtype = COMPLEX_F64 if cplx else REAL_F64
                d.device = S.device.index if S.device.index is not None else torch.cuda.current_device()
                if stream is None:
                    stream = torch.cuda.current_stream(S.device).cuda_stream
                self._keep.append(S)
        if not _is_torch(S):
            S = np.ascontiguousarray(S)
            if S.dtype not in (np.float64, np.complex128):
                S = S.astype(np.complex128 if np.iscomplexobj(S) else np.float64)
            d.S = S.ctypes.data
            d.S_mem = MEM_HOST
            d.M, d.N = S.shape
            d.ld = S.shape[1]
            d.dtype = COMPLEX_F64 if np.iscomplexobj(S) else REAL_F64
            self._keep.append(S)
        if w is not None:
            if _is_torch(w) and w.is_cuda:
                import torch
                # the library reads N doubles from the pointer: hand it a float64, contiguous
                # (N,) tensor on S's device (a converted copy is kept alive with the context)
                if w.dim() != 1 or w.shape[0] != d.N:
                    raise ValueError("w must have N entries")
                dev = torch.device("cuda", d.device) if d.S_mem == MEM_DEVICE else w.device
                w = w.to(device=dev, dtype=torch.float64).contiguous()
                d.w = w.data_ptr()
                d.w_mem = MEM_DEVICE
            else:
                wn = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
                if wn.shape != (d.N,):
                    raise ValueError("w must have N entries")
                d.w = wn.ctypes.data
                d.w_mem = MEM_HOST
            self._keep.append(w)
        d.tol = float(tol)
        d.k_max = int(k_max)
        # an explicit handle 0 is the legacy default stream (cudaStreamLegacy = 0x1); a NULL
        # stream in the descriptor would make the library create its own stream
        d.stream = None if stream is None else (1 if int(stream) == 0 else int(stream))
        d.check_finite = 1 if check_finite else 0
        d.ortho = ORTHO[ortho]
        d.residual = RESIDUAL[residual]
        d.comm = comm
        d.peer_timeout_ms = int(peer_timeout_ms)
        d.rank = rank
        d.world = world
        d.col_offset = col_offset
        d.M_global = M_global
        if nccl_id is not None:
            ctypes.memmove(d.nccl_id, nccl_id, 128)
        self.N, self.M = int(d.N), int(d.M)
        self.M_global = int(d.M_global) if d.M_global else int(d.M)
        self.cplx = d.dtype == COMPLEX_F64
        self.k_max = int(k_max)
        h = ctypes.c_void_p()
        _check(L.rbg_create_ex(ctypes.byref(h), ctypes.byref(d)))
        self.h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            lib().rbg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- execution
    def run(self):
        _check(lib().rbg_run(self.h))
        return self

    def step(self, n: int):
        _check(lib().rbg_step(self.h, int(n)))

    def sync(self):
        _check(lib().rbg_sync(self.h))

    def set_timing(self, on: bool):
        _check(lib().rbg_set_timing(self.h, 1 if on else 0))

    def set_graph_batch(self, batch: int):
        _check(lib().rbg_set_graph_batch(self.h, int(batch)))

    def iter_local(self):
        _check(lib().rbg_iter_local(self.h))

    def iter_finish(self):
        _check(lib().rbg_iter_finish(self.h))

    # -- results
    def info(self) -> tuple[int, int, str]:
        k, m, why = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _check(lib().rbg_result_info(self.h, ctypes.byref(k), ctypes.byref(m), ctypes.byref(why)))
        return k.value, m.value, STOP[why.value]

    def pivots(self) -> np.ndarray:
        k = self.info()[0]
        out = np.zeros(max(k, 1), np.int64)
        _check(lib().rbg_get_pivots(self.h, out.ctypes.data))
        return out[:k]

    def errors(self) -> np.ndarray:
        k, _, why = self.info()
        n = k + 1 if why not in ("NONE", "PEER_TIMEOUT") else k   # err_k exists once decided
        out = np.zeros(max(n, 1))
        _check(lib().rbg_get_errors(self.h, out.ctypes.data))
        return out[:n]

    def nu(self) -> np.ndarray:
        k = self.info()[0]
        out = np.zeros(max(k, 1), np.int32)
        _check(lib().rbg_get_nu(self.h, out.ctypes.data))
        return out[:k]

    def rdiag(self) -> np.ndarray:
        k = self.info()[0]
        out = np.zeros(max(k, 1))
        _check(lib().rbg_get_rdiag(self.h, out.ctypes.data))
        return out[:k]

    def basis(self) -> np.ndarray:
        k = self.info()[0]
        out = _host_out((max(k, 1), self.N), np.complex128 if self.cplx else np.float64)
        _check(lib().rbg_get_basis(self.h, out.ctypes.data, self.N, 0))
        return out[:k]

    def R(self) -> np.ndarray:
        k = self.info()[0]
        out = _host_out((max(k, 1), self.M), np.complex128 if self.cplx else np.float64)
        _check(lib().rbg_get_R(self.h, out.ctypes.data, self.M, 0))
        return out[:k]

    def r2(self) -> np.ndarray:
        out = np.zeros(self.M)
        _check(lib().rbg_get_r2(self.h, out.ctypes.data, 0))
        return out

    def stats(self) -> Stats:
        s = Stats()
        _check(lib().rbg_get_stats(self.h, ctypes.byref(s)))
        return s

    def timings(self, n: int):
        a, b, c = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(lib().rbg_get_timings(self.h, a.ctypes.data, b.ctypes.data, c.ctypes.data, n))
        return a, b, c

    def _block(self, X):
        """(pointer, M_b, ld, mem, keepalive) of an (M_b, N) host array or CUDA tensor."""
        if _is_torch(X) and X.is_cuda:
            if X.dim() != 2 or X.stride(1) != 1 or X.shape[1] != self.N:
                raise ValueError("block must be (M_b, N) with contiguous rows")
            return X.data_ptr(), X.shape[0], X.stride(0), MEM_DEVICE, X
        if _is_torch(X):
            X = X.numpy()
        X = np.ascontiguousarray(X, dtype=np.complex128 if self.cplx else np.float64)
        if X.ndim != 2 or X.shape[1] != self.N:
            raise ValueError("block must be (M_b, N)")
        return X.ctypes.data, X.shape[0], X.shape[1], MEM_HOST, X

    def validate(self, V, coeffs: bool = False):
        """Projection errors (and optionally coefficients) of the columns of V (M_v, N)
        against the current basis (rbg_validate)."""
        ptr, mv, ld, mem, keep = self._block(V)
        k = self.info()[0]
        err = np.zeros(mv)
        C = np.zeros((max(k, 1), mv), np.complex128 if self.cplx else np.float64) if coeffs else None
        _check(lib().rbg_validate(self.h, ptr, mv, ld, mem, err.ctypes.data,
                                  C.ctypes.data if coeffs else None, mv, 0))
        del keep
        return (err, C[:k]) if coeffs else err

    def add_columns(self, F, first_gid: int | None = None, M_global: int | None = None):
        """Append the columns of F (M_f, N) to the training set: rbg_add_columns on one GPU,
        rbg_add_columns_ex with their global ids (first_gid..) and the new total M_global on
        a sharded context (F may have 0 rows there)."""
        if F is None or (hasattr(F, "shape") and F.shape[0] == 0):
            ptr, mf, ld, mem, keep = None, 0, self.N, MEM_HOST, None
        else:
            ptr, mf, ld, mem, keep = self._block(F)
        if first_gid is None and M_global is None:
            _check(lib().rbg_add_columns(self.h, ptr, mf, ld, mem))
        else:
            _check(lib().rbg_add_columns_ex(self.h, ptr, mf, ld, mem, -1 if first_gid is None else int(first_gid),
                                            0 if M_global is None else int(M_global)))
        self.M += mf
        self.M_global = int(M_global) if M_global is not None else self.M_global + mf
        del keep

    def restore(self, state: "Result"):
        """rbg_restore: continue a checkpointed greedy (a Result from result(full=True) of a
        stopped context over the same S and w) in this fresh context; the next run() begins at
        the decision for state.k."""
        k = int(state.k)
        dt = np.complex128 if self.cplx else np.float64
        piv = np.ascontiguousarray(state.pivots[:k], dtype=np.int64)
        err = np.ascontiguousarray(np.asarray(state.errors)[:k], dtype=np.float64)
        nu = np.ascontiguousarray(state.nu[:k], dtype=np.int32)
        rd = np.ascontiguousarray(state.rdiag[:k], dtype=np.float64)
        Q = np.ascontiguousarray(state.Q[:k], dtype=dt)
        R = np.ascontiguousarray(state.R[:k], dtype=dt)
        r2 = np.ascontiguousarray(state.r2, dtype=np.float64)
        if Q.shape != (k, self.N) or R.shape != (k, self.M) or r2.shape != (self.M,):
            raise ValueError("checkpoint shapes do not match this context")
        _check(lib().rbg_restore(self.h, k, piv.ctypes.data, err.ctypes.data, nu.ctypes.data, rd.ctypes.data,
                                 Q.ctypes.data, self.N, R.ctypes.data, self.M, r2.ctypes.data, MEM_HOST))

    def gram(self) -> np.ndarray:
        """G = R R^H of the current coefficient block (k x k complex), rbg_gram."""
        k = self.info()[0]
        buf = np.zeros(k * k, np.complex128)        # column-major k x k
        if k:
            _check(lib().rbg_gram(self.h, buf.ctypes.data, k, 0))
        return buf.reshape((k, k), order="F")

    def reconstruct(self, tau2: float = 0.0, kr_max: int = 0):
        """Algorithm 4: (sigma (k,), kr, X (kr, N)) via rbg_reconstruct."""
        k = self.info()[0]
        sigma = np.zeros(max(k, 1))
        X = _host_out((max(k, 1), self.N), np.complex128 if self.cplx else np.float64)
        kr = ctypes.c_int64()
        _check(lib().rbg_reconstruct(self.h, float(tau2), int(kr_max), ctypes.byref(kr), sigma.ctypes.data,
                                     X.ctypes.data, self.N, 0))
        return sigma[:k], kr.value, X[:kr.value]

    def gram_fold(self, G: np.ndarray | None = None) -> np.ndarray:
        """G + R_loc R_loc^H (rbg_gram_fold): fold this rank's coefficient block onto the
        running Gram sum of the previous ranks (None = zeros, rank 0)."""
        k = self.info()[0]
        buf = (np.zeros((k, k), np.complex128, order="F") if G is None
               else np.array(G, dtype=np.complex128, order="F", copy=True))   # column-major k x k
        if buf.shape != (k, k):
            raise ValueError(f"G must be {k} x {k}")
        if k:
            _check(lib().rbg_gram_fold(self.h, buf.ctypes.data, k, 0))
        return buf

    def reconstruct_gram(self, G: np.ndarray, tau2: float = 0.0, kr_max: int = 0):
        """Algorithm 4 from a given Gram matrix (rbg_reconstruct_gram): (sigma, kr, X)."""
        k = self.info()[0]
        Gf = np.asfortranarray(G, dtype=np.complex128)
        sigma = np.zeros(max(k, 1))
        X = _host_out((max(k, 1), self.N), np.complex128 if self.cplx else np.float64)
        kr = ctypes.c_int64()
        _check(lib().rbg_reconstruct_gram(self.h, Gf.ctypes.data, k, 0, float(tau2), int(kr_max), ctypes.byref(kr),
                                          sigma.ctypes.data, X.ctypes.data, self.N, 0))
        return sigma[:k], kr.value, X[:kr.value]

    def eim(self):
        """Greedy EIM nodes of the current basis: (nodes (k,), B = Q(nodes, :) (k, k))."""
        k = self.info()[0]
        nodes = np.zeros(max(k, 1), np.int64)
        buf = np.zeros(max(k, 1) ** 2, np.complex128)
        if k:
            _check(lib().rbg_eim(self.h, nodes.ctypes.data, buf.ctypes.data, k, 0))
        B = buf[:k * k].reshape((k, k), order="F")
        return nodes[:k], (B if self.cplx else B.real.copy())

    def peer_export(self) -> bytes:
        """This rank's CUDA-IPC handles for the PEER exchange (rbg_peer_export)."""
        buf = (ctypes.c_uint8 * PEER_HANDLE_BYTES)()
        _check(lib().rbg_peer_export(self.h, buf))
        return bytes(buf)

    def peer_connect(self, handles: list[bytes]):
        """Map every rank's PEER buffers; ``handles[p]`` = rank p's peer_export()."""
        blob = b"".join(handles)
        if len(blob) != PEER_HANDLE_BYTES * len(handles):
            raise ValueError("each handle blob must be PEER_HANDLE_BYTES long")
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(lib().rbg_peer_connect(self.h, buf))

    def xchg_buffers(self):
        s, r, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().rbg_xchg_buffers(self.h, ctypes.byref(s), ctypes.byref(r), ctypes.byref(n)))
        return s.value, r.value, n.value

    def result(self, full: bool = True) -> Result:
        k, _, why = self.info()
        return Result(k=k, stop=why, pivots=self.pivots(), errors=self.errors(), nu=self.nu(),
                      rdiag=self.rdiag(), Q=self.basis() if full else None,
                      R=self.R() if full else None, r2=self.r2() if full else None)


def _rows(V, mask: np.ndarray):
    """The rows of V selected by a host boolean mask (gathered on V's device)."""
    if _is_torch(V):
        import torch
        return V[torch.as_tensor(np.nonzero(mask)[0], device=V.device)]
    return V[mask]


def enrich(ctx: Context, V, tol: float, rounds: int = 3):
    """Iterative refinement (SPEC enrich): validate V against the basis,
    append every failing column (err >= tol) not appended before, continue the greedy, and
    repeat up to `rounds` times.  A CUDA tensor V stays on the device: it is validated in
    place and its failing columns are gathered on the device.  Returns (per-round max
    validation error, passed)."""
    Vh = V if (_is_torch(V) and V.is_cuda) else (V.cpu().numpy() if _is_torch(V) else np.asarray(V))
    added = np.zeros(Vh.shape[0], bool)
    history = []
    for _ in range(rounds):
        err = ctx.validate(Vh)
        history.append(float(err.max()) if err.size else 0.0)
        fail = (err >= tol) & ~added
        if not fail.any():
            return history, bool(np.all(err < tol))
        ctx.add_columns(_rows(Vh, fail))
        added |= fail
        ctx.run()
    err = ctx.validate(Vh)
    history.append(float(err.max()) if err.size else 0.0)
    return history, bool(np.all(err < tol))


def peer_connect_local(ctxs: list[Context]):
    """Wire PEER contexts of this process (one device, one stream) to each other (tests)."""
    arr = (ctypes.c_void_p * len(ctxs))(*[c.h for c in ctxs])
    _check(lib().rbg_peer_connect_local(arr, len(ctxs)))


def emulate_allgather(ctxs: list[Context]):
    arr = (ctypes.c_void_p * len(ctxs))(*[c.h for c in ctxs])
    _check(lib().rbg_emulate_allgather(arr, len(ctxs)))


def greedy(S, w=None, tol: float = 0.0, k_max: int = 1, full: bool = True, **kw) -> Result:
    """Run the RB-greedy to its stop reason on one GPU and return the results (host)."""
    with Context(S, w, tol, k_max, **kw) as ctx:
        ctx.run()
        return ctx.result(full)


def gen_chirp(S, t, w, q, chi, psi, spin: bool, stream=None):
    """Fill the CUDA complex128 tensor S (M, N) with chirps on the device (rbg_gen.h)."""
    import torch
    from .inputs import CHIRP_EPS, CHIRP_F0
    dev = S.device
    x = (-np.asarray(t) + CHIRP_EPS)
    A = torch.as_tensor(x ** -0.25, device=dev)
    base = torch.as_tensor(-2.0 * np.pi * CHIRP_F0 * x ** 0.625 / 0.625, device=dev)
    wt = torch.as_tensor(np.asarray(w, dtype=np.float64), device=dev)
    qt = torch.as_tensor(np.asarray(q, dtype=np.float64), device=dev)
    ct = torch.as_tensor(np.asarray(chi, dtype=np.float64), device=dev)
    pt = torch.as_tensor(np.asarray(psi, dtype=np.float64), device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    M, N = S.shape
    rc = lib().rbg_gen_chirp(S.data_ptr(), N, M, S.stride(0), A.data_ptr(), base.data_ptr(),
                             wt.data_ptr(), qt.data_ptr(), ct.data_ptr(), pt.data_ptr(),
                             1 if spin else 0, stream)
    if rc != 0:
        raise RbgError(ECUDA, f"rbg_gen_chirp failed ({rc})")
    torch.cuda.current_stream(dev).synchronize()
    del A, base, wt, qt, ct, pt


# ----------------------------------------------------------------------------- C-ABI names
# One Python function per entry point of include/rbg.h, named as the C function without its
# `rbg_` prefix (argument marshalling only; tests/test_abi.py checks the correspondence).

def create(S, N: int | None = None, M: int | None = None, w=None, tol: float = 0.0, k_max: int = 1,
           dtype=None) -> Context:
    """rbg_create: host S (M, N) array (N, M, dtype are implied by the array)."""
    return Context(np.asarray(S), w, tol, k_max)


def create_ex(S, w=None, tol: float = 0.0, k_max: int = 1, **kw) -> Context:
    """rbg_create_ex: host array or CUDA tensor, plus the rbg_desc fields as keywords."""
    return Context(S, w, tol, k_max, **kw)


def desc_init() -> Desc:
    """rbg_desc_init: a descriptor with the library defaults."""
    d = Desc()
    lib().rbg_desc_init(ctypes.byref(d))
    return d


def get_unique_id() -> bytes:
    return unique_id()


def run(ctx: Context):
    return ctx.run()


def step(ctx: Context, n: int):
    ctx.step(n)


def set_timing(ctx: Context, on: bool):
    ctx.set_timing(on)


def set_graph_batch(ctx: Context, batch: int):
    ctx.set_graph_batch(batch)


def sync(ctx: Context):
    ctx.sync()


def result_info(ctx: Context) -> tuple[int, int, str]:
    return ctx.info()


def get_pivots(ctx: Context) -> np.ndarray:
    return ctx.pivots()


def get_errors(ctx: Context) -> np.ndarray:
    return ctx.errors()


def get_nu(ctx: Context) -> np.ndarray:
    return ctx.nu()


def get_rdiag(ctx: Context) -> np.ndarray:
    return ctx.rdiag()


def get_basis(ctx: Context) -> np.ndarray:
    return ctx.basis()


def get_R(ctx: Context) -> np.ndarray:  # noqa: N802 (C name)
    return ctx.R()


def get_r2(ctx: Context) -> np.ndarray:
    return ctx.r2()


def get_stats(ctx: Context) -> Stats:
    return ctx.stats()


def get_timings(ctx: Context, n: int):
    return ctx.timings(n)


def validate(ctx: Context, V, coeffs: bool = False):
    return ctx.validate(V, coeffs)


def add_columns(ctx: Context, F):
    ctx.add_columns(F)


def add_columns_ex(ctx: Context, F, first_gid: int, M_global: int):
    ctx.add_columns(F, first_gid=first_gid, M_global=M_global)


def gram(ctx: Context) -> np.ndarray:
    return ctx.gram()


def restore(ctx: Context, state: Result):
    ctx.restore(state)


def save_checkpoint(ctx: Context, path: str):
    """The stopped greedy's state (the getters' outputs) as an .npz file."""
    r = ctx.result(full=True)
    np.savez(path, k=r.k, stop=r.stop, pivots=r.pivots, errors=r.errors, nu=r.nu, rdiag=r.rdiag, Q=r.Q, R=r.R, r2=r.r2)


def load_checkpoint(path: str) -> Result:
    z = np.load(path)
    return Result(k=int(z["k"]), stop=str(z["stop"]), pivots=z["pivots"], errors=z["errors"], nu=z["nu"],
                  rdiag=z["rdiag"], Q=z["Q"], R=z["R"], r2=z["r2"])


def gram_fold(ctx: Context, G=None) -> np.ndarray:
    return ctx.gram_fold(G)


def reconstruct(ctx: Context, tau2: float = 0.0, kr_max: int = 0):
    return ctx.reconstruct(tau2, kr_max)


def reconstruct_gram(ctx: Context, G, tau2: float = 0.0, kr_max: int = 0):
    return ctx.reconstruct_gram(G, tau2, kr_max)


def eim(ctx: Context):
    return ctx.eim()


def iter_local(ctx: Context):
    ctx.iter_local()


def iter_finish(ctx: Context):
    ctx.iter_finish()


def xchg_buffers(ctx: Context):
    return ctx.xchg_buffers()


def peer_export(ctx: Context) -> bytes:
    return ctx.peer_export()


def peer_connect(ctx: Context, handles: list[bytes]):
    ctx.peer_connect(handles)


def debug_set_canary(on: bool):
    set_canary(on)


def debug_canary_violations() -> tuple[int, str]:
    return canary_violations()


def last_error() -> str:
    return lib().rbg_last_error().decode()


def destroy(ctx: Context):
    ctx.close()
