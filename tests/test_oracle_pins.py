"""Pins of the CPU oracle against what arXiv 1805.06124 and mathematics fix.

None of these retypes the oracle's formula: each compares it with a closed form, a
theorem of the paper evaluated by brute force, an independent algorithm of the paper
(Algorithm 2), a library special case (LAPACK xGEQP3, numpy vdot/SVD), or exact
rational arithmetic.  Both lane modes (plain (1,1) and canonical (32,2048)) are pinned.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.linalg

import brute
from paper_1805_06124_b200 import inputs

MODES = [(1, 1), (32, 2048), (4, 8)]


def rand_matrix(rng, N, M, cplx=True, rank=None):
    if rank is None:
        A = rng.standard_normal((M, N))
        if cplx:
            A = A + 1j * rng.standard_normal((M, N))
        return A
    L = rng.standard_normal((M, rank))
    Rt = rng.standard_normal((rank, N))
    if cplx:
        L = L + 1j * rng.standard_normal((M, rank))
        Rt = Rt + 1j * rng.standard_normal((rank, N))
    return L @ Rt


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("lanes", MODES)
def test_identity_matrix(orc, lanes):
    r = orc.greedy(np.eye(3), np.ones(3), 0.0, 3, lanes=lanes)
    assert r.k == 3 and r.stop == "ALL_SELECTED"
    assert list(r.pivots) == [0, 1, 2]               # lowest index on ties (reading R9)
    assert list(r.errors) == [1.0, 1.0, 1.0, 0.0]
    np.testing.assert_array_equal(r.Q, np.eye(3))
    np.testing.assert_array_equal(r.R, np.eye(3))


@pytest.mark.parametrize("lanes", MODES)
def test_diagonal_matrix(orc, lanes):
    r = orc.greedy(np.diag([3.0, 2.0, 1.0]), np.ones(3), 0.0, 3, lanes=lanes)
    assert list(r.pivots) == [0, 1, 2]
    assert list(r.errors) == [3.0, 2.0, 1.0, 0.0]
    assert list(r.rdiag) == [3.0, 2.0, 1.0]


def test_two_columns(orc):
    S = np.array([[2.0, 0.0], [0.0, 1.0]])            # rows = columns (2 e1, e2)
    r = orc.greedy(S, np.ones(2), 0.0, 2)
    assert list(r.pivots) == [0, 1] and list(r.errors) == [2.0, 1.0, 0.0]
    assert r.stop == "ALL_SELECTED"


def test_tolerance_and_kmax_stops(orc):
    S = np.diag([3.0, 2.0, 1.0])
    r = orc.greedy(S, np.ones(3), 1.5, 3)              # err_2 = 1 < 1.5 -> TOL at k=2
    assert (r.k, r.stop, list(r.errors)) == (2, "TOL", [3.0, 2.0, 1.0])
    r = orc.greedy(S, np.ones(3), 2.0, 3)              # err_1 = 2 is not < 2 (Algo 3 uses >=)
    assert (r.k, r.stop) == (2, "TOL")
    r = orc.greedy(S, np.ones(3), 0.0, 2)
    assert (r.k, r.stop, list(r.errors)) == (2, "KMAX", [3.0, 2.0, 1.0])


def test_zero_matrix_is_rank_stop(orc):
    r = orc.greedy(np.zeros((4, 5)), np.ones(5), 0.0, 3)
    assert r.k == 0 and r.stop == "RANK" and list(r.errors) == [0.0]


@pytest.mark.parametrize("lanes", MODES)
def test_orthogonal_columns_descending_norm(orc, lanes):
    """Mutually W-orthogonal columns are picked in descending norm order, ties -> lowest."""
    # Sylvester-Hadamard columns divided by sqrt(w_i) in {1/2, 1, 2}: exactly W-orthogonal
    # in floating point, so equal norms are exact ties.
    rng = np.random.default_rng(7)
    N, M = 16, 10
    H = np.array([[1.0]])
    while H.shape[0] < N:
        H = np.block([[H, H], [H, -H]])
    w = rng.choice([0.25, 1.0, 4.0], N)
    ph = rng.choice([1, -1, 1j, -1j], M)
    scale = np.array([3.0, 5.0, 5.0, 1.0, 7.0, 2.0, 5.0, 0.5, 4.0, 6.0])
    S = (H[:, :M] / np.sqrt(w)[:, None] * (scale * ph)[None, :]).T / 4.0
    r = orc.greedy(S, w, 0.0, M, lanes=lanes)
    expect = sorted(range(M), key=lambda j: (-scale[j], j))
    assert list(r.pivots) == expect
    np.testing.assert_array_equal(r.errors[:M], scale[expect])


# ---------------------------------------------------------------- the canonical dot (error bound)

@pytest.mark.parametrize("L", [1, 2, 32, 2048])
@pytest.mark.parametrize("cplx", [False, True])
def test_dot_within_higham_bound(orc, L, cplx):
    """|DOT_L - exact| <= gamma_m sum |x~_i||y_i| with m = chain length + log2 L + 2."""
    rng = np.random.default_rng(11 + L)
    n = 301
    x = rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0)
    y = rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0)
    got = orc.dot(x, y, L)
    ex_re, ex_im = brute.exact_dot(x, y)
    V = 1 if cplx else 2
    chain = 2 * math.ceil(n / (V * L)) * V
    m = chain + int(math.log2(L)) + 2
    u = 2.0 ** -53
    gamma = m * u / (1 - m * u)
    bound = gamma * float(np.sum(np.abs(x) * np.abs(y))) * 2
    g = complex(got)
    assert abs(g.real - float(ex_re)) <= bound
    assert abs(g.imag - float(ex_im)) <= bound
    # and it is the conjugate-linear product numpy.vdot defines (operand order pinned)
    ref = np.vdot(x, y)
    assert abs(g - ref) <= 2 * bound


@pytest.mark.parametrize("L", [1, 32, 2048])
def test_nrm_weighted(orc, L):
    rng = np.random.default_rng(3)
    n = 257
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    w = rng.uniform(0.5, 1.5, n)
    got = orc.nrm(y, w, L)
    exact = sum(float(w[i]) * (y[i].real ** 2 + y[i].imag ** 2) for i in range(n))
    assert abs(got - exact) <= 1e-13 * exact
    yr = y.real.copy()
    assert abs(orc.nrm(yr, w, L) - float(np.sum(w * yr * yr))) <= 1e-13 * float(np.sum(w * yr * yr))


def test_lane_counts_beyond_length_change_nothing(orc):
    """Empty lanes add +0: L = 2048 and L = 4096 agree bit for bit when n <= 2048."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal(500) + 1j * rng.standard_normal(500)
    y = rng.standard_normal(500) + 1j * rng.standard_normal(500)
    assert orc.dot(x, y, 2048) == orc.dot(x, y, 4096) == orc.dot(x, y, 512)


# ---------------------------------------------------------------- IMGS

def test_imgs_spec_examples(orc):
    q, coeff, n, nu = orc.imgs(np.zeros((0, 3)), np.array([2.0, 0.0, 0.0]), np.ones(3))
    assert list(q) == [1.0, 0.0, 0.0] and nu == 1 and n == 2.0 and coeff.size == 0
    q, coeff, n, nu = orc.imgs(np.array([[1.0, 0.0, 0.0]]), np.array([1.0, 1.0, 0.0]), np.ones(3))
    np.testing.assert_allclose(q, [0.0, 1.0, 0.0], atol=1e-14)
    np.testing.assert_allclose(coeff, [1.0], atol=1e-14)


@pytest.mark.parametrize("L", [1, 2048])
def test_imgs_orthogonality_and_reconstruction(orc, L):
    rng = np.random.default_rng(21)
    N, k = 1000, 50
    w = rng.uniform(0.5, 1.5, N)
    Q = np.zeros((0, N), np.complex128)
    for _ in range(k):
        v = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        q, coeff, n, nu = orc.imgs(Q, v, w, L)
        # v = Q coeff + n q
        rec = (Q.T @ coeff if len(coeff) else 0) + n * q
        assert np.sqrt(np.sum(w * np.abs(v - rec) ** 2)) <= 1e-12 * np.sqrt(np.sum(w * np.abs(v) ** 2))
        assert 1 <= nu <= 3
        Q = np.vstack([Q, q])
    G = (Q.conj() * w[None, :]) @ Q.T
    assert np.max(np.abs(G - np.eye(k))) <= 1e-13


def test_imgs_degenerate(orc):
    rng = np.random.default_rng(2)
    N = 40
    w = np.ones(N)
    Q = np.linalg.qr(rng.standard_normal((N, 5)))[0].T
    v = Q.T @ rng.standard_normal(5)                  # in span(Q)
    assert orc.imgs(Q, v, w) is None
    assert orc.imgs(Q, np.zeros(N), w) is None


# ---------------------------------------------------------------- equivalence theorems

@pytest.mark.parametrize("lanes", MODES)
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_prop55_and_xgeqp3(orc, lanes, cplx, seed):
    """Prop. 5.5: Algorithm 2 gives the same pivots; LAPACK xGEQP3 on
    W^{1/2}S gives the same pivots with |diag R| = err_k; Q and |R| agree with both."""
    rng = np.random.default_rng(100 + seed)
    N, M, K = 30, 80, 20
    S = rand_matrix(rng, N, M, cplx)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K, lanes=lanes)
    assert r.k == K and r.stop == "KMAX"
    St = brute.weighted(S, w)
    piv2, rd2, Q2, R2 = brute.mgs_pivoting(St, K)
    np.testing.assert_array_equal(r.pivots, piv2)
    np.testing.assert_allclose(r.errors[:K], rd2, rtol=1e-12)
    np.testing.assert_allclose(r.rdiag, rd2, rtol=1e-12)
    Ql, Rl, P = scipy.linalg.qr(St, pivoting=True, mode="economic")
    np.testing.assert_array_equal(r.pivots, P[:K])
    np.testing.assert_allclose(r.errors[:K], np.abs(np.diag(Rl))[:K], rtol=1e-12)
    # basis: W^{1/2} q_i equals the LAPACK column up to a unit phase
    Qt = (np.sqrt(w)[None, :] * r.Q).T
    ph = np.sum(Ql[:, :K].conj() * Qt, axis=0)
    np.testing.assert_allclose(np.abs(ph), 1.0, atol=1e-12)
    np.testing.assert_allclose(Qt, Ql[:, :K] * ph[None, :], atol=1e-12)
    # R: row i of the sweep coefficients equals LAPACK's row i (pivoted order) times conj phase
    Rp = r.R[:, P]
    np.testing.assert_allclose(Rp[:K, K:], (ph.conj()[:, None] * Rl[:K, K:]), atol=1e-11)
    # and Algorithm 2's coefficients on the non-pivot columns of the first row
    np.testing.assert_allclose(np.abs(r.R[0]), np.abs(R2[0]), atol=1e-12)


@pytest.mark.parametrize("lanes", [(1, 1), (32, 2048)])
def test_cor56_stop_identity_and_monotone(orc, lanes):
    """Cor. 5.6: err_k = max_j ||(I - P_k) s~_j|| (direct projection),
    = R(k+1,k+1) (the IMGS norm), and errors are non-increasing (Prop. 5.5 eq. Rprop)."""
    rng = np.random.default_rng(9)
    N, M, K = 40, 120, 25
    S = rand_matrix(rng, N, M, True)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K, lanes=lanes)
    St = brute.weighted(S, w)
    scale = np.max(np.sqrt(np.sum(np.abs(St) ** 2, axis=0)))
    for k in range(K + 1):
        Qt = (np.sqrt(w)[None, :] * r.Q[:k]).T
        d = brute.direct_residuals(St, Qt)
        assert abs(d.max() - r.errors[k]) <= 1e-10 * scale
        if k < K:
            assert int(np.argmax(d)) == r.pivots[k]
            assert abs(r.rdiag[k] - r.errors[k]) <= 1e-10 * scale
    assert np.all(np.diff(r.errors) <= 1e-12 * scale)


def test_thm42_residual_consistency(orc):
    """Thm. 4.2: ||s_j||^2 - sum_i |R(i,j)|^2 = r2_j; R11 upper
    triangular; full-rank run reconstructs S = Q R."""
    rng = np.random.default_rng(4)
    N, M = 16, 40
    S = rand_matrix(rng, N, M, True)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, 10)
    nrm2 = np.sum(w[None, :] * np.abs(S) ** 2, axis=1)
    unsel = np.setdiff1d(np.arange(M), r.pivots)
    lhs = nrm2 - np.sum(np.abs(r.R) ** 2, axis=0)
    np.testing.assert_allclose(lhs[unsel], r.r2[unsel], atol=1e-12 * nrm2.max())
    R11 = r.R[:, r.pivots]
    assert np.max(np.abs(np.tril(R11, -1))) <= 1e-13 * nrm2.max()
    r = orc.greedy(S, w, 0.0, N)                        # full numerical rank N
    Srec = r.Q.T @ r.R                                  # N x M
    np.testing.assert_allclose(Srec, S.T, atol=1e-12 * np.sqrt(nrm2.max()))


@pytest.mark.parametrize("cplx", [False, True])
def test_cor57_volume_identity(orc, cplx):
    """Cor. 5.7, reading R4: prod sigma_i(S~_{k+1}) = prod R(i,i) over
    the first k+1 pivoted columns; sigma by one-sided Jacobi (checked against LAPACK)."""
    rng = np.random.default_rng(12)
    N, M, K = 20, 30, 8
    S = rand_matrix(rng, N, M, cplx)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K)
    St = brute.weighted(S, w)
    for k in range(1, K):
        sub = St[:, r.pivots[: k + 1]]
        sv = brute.jacobi_svd_values(sub)
        np.testing.assert_allclose(sv, np.linalg.svd(sub, compute_uv=False), rtol=1e-12)
        assert abs(np.sum(np.log(sv)) - np.sum(np.log(r.errors[: k + 1]))) <= 1e-8


def test_sigma_bounds(orc):
    """Reading R16: ||(I-P_k) S~||_2 >= sigma_{k+1}(S~) (Thm 3.2 / Remark)
    and sigma_{k+1}/sqrt(M-k) <= err_k <= ||(I-P_k) S~||_2 (Cor. 4.3)."""
    rng = np.random.default_rng(13)
    N, M, K = 24, 36, 12
    S = rand_matrix(rng, N, M, True)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K)
    St = brute.weighted(S, w)
    sig = brute.jacobi_svd_values(St)
    for k in range(K + 1):
        Qt = (np.sqrt(w)[None, :] * r.Q[:k]).T
        E = St - Qt @ (Qt.conj().T @ St) if k else St
        e2 = np.linalg.norm(E, 2)
        assert e2 >= sig[k] * (1 - 1e-12)
        assert sig[k] / np.sqrt(M - k) <= r.errors[k] * (1 + 1e-12)
        assert r.errors[k] <= e2 * (1 + 1e-12)


def test_scaling_and_phase_invariance(orc):
    rng = np.random.default_rng(14)
    N, M, K = 32, 64, 16
    S = rand_matrix(rng, N, M, True)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K)
    r8 = orc.greedy(S * 8.0, w, 0.0, K)                # power of two: exact scaling
    np.testing.assert_array_equal(r8.pivots, r.pivots)
    np.testing.assert_array_equal(r8.errors, 8.0 * r.errors)
    r3 = orc.greedy(S * 3.0, w, 0.0, K)
    np.testing.assert_array_equal(r3.pivots, r.pivots)
    np.testing.assert_allclose(r3.errors, 3.0 * r.errors, rtol=1e-12)
    th = rng.uniform(0, 2 * np.pi, M)
    rp = orc.greedy(S * np.exp(1j * th)[:, None], w, 0.0, K)
    np.testing.assert_array_equal(rp.pivots, r.pivots)
    np.testing.assert_allclose(rp.errors, r.errors, rtol=1e-12)
    # R rows rotate with the column phases (and q_i picks up the pivot's phase)
    ph_q = np.exp(1j * th[r.pivots])
    np.testing.assert_allclose(rp.R, (ph_q.conj()[:, None] * r.R * np.exp(1j * th)[None, :]),
                               atol=1e-11)


def test_orthonormality(orc):
    S, w, tol, k_max = inputs.config1(M=600, N=400)
    r = orc.greedy(S, w, tol, k_max)
    G = (r.Q.conj() * w[None, :]) @ r.Q.T
    assert np.max(np.abs(G - np.eye(r.k))) <= 1e-12


def test_exact_rank_stops_at_rank(orc):
    """An exactly rank-r input (well conditioned) stops RANK at k = r (reading R17)."""
    rng = np.random.default_rng(15)
    for cplx, r_ in [(False, 7), (True, 11)]:
        S = rand_matrix(rng, 50, 90, cplx, rank=r_)
        res = orc.greedy(S, np.ones(50), 0.0, 50)
        assert res.k == r_ and res.stop == "RANK"


def test_thread_count_invariance(orc):
    S, w, tol, k_max = inputs.config0()
    a = orc.greedy(S, w, tol, k_max, threads=1)
    b = orc.greedy(S, w, tol, k_max, threads=8)
    np.testing.assert_array_equal(a.pivots, b.pivots)
    np.testing.assert_array_equal(a.Q, b.Q)
    np.testing.assert_array_equal(a.R, b.R)
    np.testing.assert_array_equal(a.errors, b.errors)


def test_canonical_vs_plain_agree_while_separated(orc):
    """Both lane modes are valid orders; on cfg0 they agree on every pivot while the
    residual gap is far above the rounding level (reading R8: they diverge only in the
    recurrence's accuracy floor)."""
    S, w, tol, k_max = inputs.config0()
    a = orc.greedy(S, w, tol, k_max, lanes=(32, 2048))
    b = orc.greedy(S, w, tol, k_max, lanes=(1, 1))
    n = min(a.k, b.k)
    d = int(np.argmax(a.pivots[:n] != b.pivots[:n])) if np.any(a.pivots[:n] != b.pivots[:n]) else n
    assert a.errors[d] < 1e-5 * a.errors[0]
    # identical up to the floor scale (~sqrt(eps) * max ||s||, reading R8) ...
    np.testing.assert_allclose(a.errors[:d], b.errors[:d], rtol=0, atol=1e-7 * a.errors[0])
    # ... and the squared residuals (the recurrence's own variable) to ~1e4 eps * max ||s||^2
    np.testing.assert_allclose(a.errors[:d] ** 2, b.errors[:d] ** 2, rtol=0,
                               atol=1e-12 * a.errors[0] ** 2)


# ---------------------------------------------------------------- CGSCI variant

@pytest.mark.parametrize("cplx", [False, True])
def test_cgs_variant_equivalence_and_orthogonality(orc, cplx):
    """Iterated classical GS gives the same pivots as LAPACK xGEQP3 / Algorithm 2 on
    separated inputs, |diag R| = err_k, and an orthonormal basis."""
    rng = np.random.default_rng(200)
    N, M, K = 30, 80, 20
    S = rand_matrix(rng, N, M, cplx)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K, lanes=orc.CANONICAL_CGS, ortho="cgs")
    St = brute.weighted(S, w)
    Ql, Rl, P = scipy.linalg.qr(St, pivoting=True, mode="economic")
    np.testing.assert_array_equal(r.pivots, P[:K])
    np.testing.assert_allclose(r.errors[:K], np.abs(np.diag(Rl))[:K], rtol=1e-12)
    G = (r.Q.conj() * w[None, :]) @ r.Q.T
    assert np.max(np.abs(G - np.eye(K))) <= 1e-13


def test_cgs_variant_closed_forms_and_rank(orc):
    r = orc.greedy(np.eye(3), np.ones(3), 0.0, 3, lanes=orc.CANONICAL_CGS, ortho="cgs")
    assert list(r.pivots) == [0, 1, 2] and list(r.errors) == [1.0, 1.0, 1.0, 0.0]
    rng = np.random.default_rng(201)
    S = rand_matrix(rng, 50, 90, True, rank=9)
    res = orc.greedy(S, np.ones(50), 0.0, 50, lanes=orc.CANONICAL_CGS, ortho="cgs")
    assert res.k == 9 and res.stop == "RANK"


# ---------------------------------------------------------------- explicit residuals (8f-4)

@pytest.mark.parametrize("cplx", [False, True])
def test_explicit_mode_is_algorithm2(orc, cplx):
    """Explicit residuals = Algorithm 2 (MGS with pivoting, in-place updates) + IMGS of the
    updated pivot column: same pivots as the independent Algorithm 2 and xGEQP3, |diag R|."""
    rng = np.random.default_rng(300)
    N, M, K = 30, 80, 25
    S = rand_matrix(rng, N, M, cplx)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, K, residual="explicit")
    St = brute.weighted(S, w)
    piv2, rd2, _, _ = brute.mgs_pivoting(St, K)
    np.testing.assert_array_equal(r.pivots, piv2)
    np.testing.assert_allclose(r.errors[:K], rd2, rtol=1e-12)
    Ql, Rl, P = scipy.linalg.qr(St, pivoting=True, mode="economic")
    np.testing.assert_array_equal(r.pivots, P[:K])
    G = (r.Q.conj() * w[None, :]) @ r.Q.T
    assert np.max(np.abs(G - np.eye(K))) <= 1e-13
    # R is Algorithm 2's factor: upper triangular in pivoted order, diagonal = residual norms
    R11 = r.R[:, r.pivots]
    scale = np.abs(R11).max()
    assert np.max(np.abs(np.tril(R11, -1))) <= 1e-14 * scale
    np.testing.assert_allclose(np.abs(np.diag(R11)), r.errors[:K], rtol=1e-12)


def test_explicit_mode_beats_the_recurrence_floor(orc):
    """Reading R8: the recurrence stalls near sqrt(eps) max||s|| and stops RANK on config 0;
    explicit residuals reach the paper's tolerance (Cor. 5.6 holds to ~eps, checked by direct
    projection)."""
    S, w, tol, k_max = inputs.config0()
    a = orc.greedy(S, w, tol, k_max)
    b = orc.greedy(S, w, tol, k_max, residual="explicit")
    assert a.stop == "RANK" and a.errors[-1] > 1e-9
    assert b.stop == "TOL" and b.errors[-1] < tol
    St = brute.weighted(S, w)
    scale = np.sqrt(np.max(np.sum(w * S * S, axis=1)))
    for k in (10, 40, b.k - 1, b.k):
        Qt = (np.sqrt(w)[None, :] * b.Q[:k]).T
        d = brute.direct_residuals(St, Qt)
        assert abs(d.max() - b.errors[k]) <= 1e-13 * scale
