"""Brute-force references used to PIN the oracle (tests only).

Each is written from the paper or from textbook mathematics, independently of
oracle/rbg_oracle.c, so that a dropped term, a wrong index or a transposed operand in
the oracle shows up as a disagreement.
"""
from __future__ import annotations

import ctypes
import ctypes.util
from fractions import Fraction

import numpy as np


def weighted(S_rows: np.ndarray, w: np.ndarray) -> np.ndarray:
    """S~ = W^{1/2} S as an (N, M) matrix from (M, N) rows (reading R6)."""
    return (np.sqrt(w)[None, :] * S_rows).T.copy()


def mgs_pivoting(St: np.ndarray, k_max: int, tau: float = 0.0):
    """Algorithm 2 "MGS with pivoting" with the index typo of line 9
    read as Q(:,k) (reading R1) and explicit in-place column updates V(:,j) -= R(k,j) q_k
    for every remaining column.  Column norms are recomputed from V each step.
    Returns (pivots, Rdiag, Q (N x k), Rrows (k x M))."""
    V = np.array(St, dtype=np.result_type(St.dtype, np.float64), copy=True)
    N, M = V.shape
    piv, rd, qs, rows = [], [], [], []
    for _ in range(min(k_max, M)):
        norms = np.sqrt(np.sum(np.abs(V) ** 2, axis=0))
        norms[piv] = -1.0
        i = int(np.argmax(norms))          # first maximal index on ties (reading R9)
        if norms[i] <= tau:
            break
        q = V[:, i] / norms[i]
        r = q.conj() @ V
        r[piv] = 0.0
        r[i] = norms[i]
        V = V - np.outer(q, r)
        V[:, i] = 0.0
        piv.append(i)
        rd.append(norms[i])
        qs.append(q)
        rows.append(r)
    return (np.array(piv, dtype=np.int64), np.array(rd),
            np.array(qs).T if qs else np.zeros((N, 0)), np.array(rows))


def jacobi_svd_values(A: np.ndarray, sweeps: int = 60) -> np.ndarray:
    """Singular values by one-sided (Hestenes) Jacobi rotations; descending.  Textbook
    algorithm, used on tiny matrices only."""
    U = np.array(A, dtype=np.complex128 if np.iscomplexobj(A) else np.float64, copy=True)
    if U.shape[1] > U.shape[0]:
        U = U.conj().T.copy()          # same singular values, fewer columns
    n = U.shape[1]
    for _ in range(sweeps):
        off = 0.0
        for p in range(n - 1):
            for q in range(p + 1, n):
                a = np.vdot(U[:, p], U[:, p]).real
                b = np.vdot(U[:, q], U[:, q]).real
                c = np.vdot(U[:, p], U[:, q])
                if abs(c) <= 1e-15 * np.sqrt(a * b) or a * b == 0.0:
                    continue
                off = max(off, abs(c) / np.sqrt(a * b))
                # rotate so that columns p and q become orthogonal
                phase = c / abs(c)
                zeta = (b - a) / (2.0 * abs(c))
                t = np.sign(zeta) / (abs(zeta) + np.sqrt(1.0 + zeta * zeta)) if zeta != 0 else 1.0
                cs = 1.0 / np.sqrt(1.0 + t * t)
                sn = cs * t
                up = U[:, p].copy()
                U[:, p] = cs * up - sn * np.conj(phase) * U[:, q]
                U[:, q] = sn * phase * up + cs * U[:, q]
        if off < 1e-15:
            break
    s = np.sqrt(np.sum(np.abs(U) ** 2, axis=0))
    return np.sort(s)[::-1]


def exact_dot(xt: np.ndarray, y: np.ndarray):
    """sum_i conj(xt_i) y_i in exact rational arithmetic (Fractions of the doubles)."""
    if np.iscomplexobj(xt):
        re = Fraction(0)
        im = Fraction(0)
        for a, b in zip(xt, y):
            ar, ai = Fraction(a.real), Fraction(a.imag)
            br, bi = Fraction(b.real), Fraction(b.imag)
            re += ar * br + ai * bi
            im += ar * bi - ai * br
        return re, im
    s = Fraction(0)
    for a, b in zip(xt, y):
        s += Fraction(float(a)) * Fraction(float(b))
    return s, Fraction(0)


def direct_residuals(St: np.ndarray, Qt: np.ndarray) -> np.ndarray:
    """||s~_j - Q~ Q~^H s~_j||_2 for every column, by explicit projection (Cor. 5.6)."""
    if Qt.shape[1] == 0:
        return np.sqrt(np.sum(np.abs(St) ** 2, axis=0))
    E = St - Qt @ (Qt.conj().T @ St)
    return np.sqrt(np.sum(np.abs(E) ** 2, axis=0))


_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double] * 3


def fma(a: float, b: float, c: float) -> float:
    """Correctly rounded a*b + c (C99 fma; Python 3.12 has no math.fma)."""
    return _libm.fma(a, b, c)
