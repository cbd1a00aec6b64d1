"""Algorithm 4 "Reconstruction" (Thm 5.8; Lemma 5.11 /
Thm 5.12) -- DESIGN.md NEXT f-3.

Oracle pins (CPU): the reconstructed basis of an exact-rank matrix is POD-optimal
(Thm 5.8), its singular values are those of W^{1/2}S, and the bounds of Lemma 5.11 /
Thm 5.12 hold on a truncated run.  GPU parity: the Gram matrix bit for bit, singular values
and the reconstructed basis (up to unit phases) within tolerance.
"""
import numpy as np
import pytest

import brute


def _lowrank(rng, N, M, r, cplx=True, decay=0.5):
    U = rng.standard_normal((N, r)) + (1j * rng.standard_normal((N, r)) if cplx else 0)
    V = rng.standard_normal((M, r)) + (1j * rng.standard_normal((M, r)) if cplx else 0)
    U, _ = np.linalg.qr(U)
    V, _ = np.linalg.qr(V)
    s = decay ** np.arange(r)
    return ((U * s) @ V.conj().T).T.copy()          # (M, N) rows = columns of S


def _pod_error(St, Xt, j):
    E = St - Xt[:, :j] @ (Xt[:, :j].conj().T @ St)
    return np.linalg.norm(E, 2)


@pytest.mark.parametrize("cplx", [True, False])
def test_thm58_exact_rank_is_pod_optimal(orc, cplx):
    rng = np.random.default_rng(3)
    N, M, r = 40, 60, 8
    S = _lowrank(rng, N, M, r, cplx)
    w = rng.uniform(0.5, 1.5, N)
    res = orc.greedy(S, w, 0.0, N)
    assert res.stop == "RANK" and res.k == r
    sigma, kr, X, _ = orc.reconstruct(res, 0.0)
    St = brute.weighted(S, w)
    sv = np.linalg.svd(St, compute_uv=False)
    np.testing.assert_allclose(sigma, sv[:r], rtol=1e-10)
    Xt = (np.sqrt(w)[None, :] * X).T
    np.testing.assert_allclose(Xt.conj().T @ Xt, np.eye(kr), atol=1e-12)   # W-orthonormal X
    for j in range(1, r):
        # ||S - X_j X_j^H S||_2 = sigma_{j+1} (Thm 5.8), and the POD error equals it
        assert abs(_pod_error(St, Xt, j) - sv[j]) <= 1e-10 * sv[0]


def test_truncated_run_bounds(orc):
    """Lemma 5.11 / Thm 5.12: sigma_{j+1}(S~) <= ||S~ - X_j X_j^H S~||_2 <= sigma_{j+1}(R_k) + ||R22||_2."""
    rng = np.random.default_rng(4)
    N, M = 30, 50
    S = rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))
    w = rng.uniform(0.5, 1.5, N)
    k = 12
    res = orc.greedy(S, w, 0.0, k)
    sigma, kr, X, _ = orc.reconstruct(res, 0.0)
    St = brute.weighted(S, w)
    sv = np.linalg.svd(St, compute_uv=False)
    Qt = (np.sqrt(w)[None, :] * res.Q).T
    r22 = np.linalg.norm(St - Qt @ (Qt.conj().T @ St), 2)      # ||R22||_2 = ||(I - P_k) S~||_2
    Xt = (np.sqrt(w)[None, :] * X).T
    for j in range(1, k):
        e = _pod_error(St, Xt, j)
        assert e >= sv[j] * (1 - 1e-12)
        assert e <= sigma[j] + r22 + 1e-12 * sv[0]


def test_gram_chunk_order_and_tau2(orc):
    rng = np.random.default_rng(5)
    R = rng.standard_normal((9, 10000)) + 1j * rng.standard_normal((9, 10000))
    G = orc.gram(R)
    np.testing.assert_allclose(G, R @ R.conj().T, rtol=0, atol=1e-13 * np.abs(G).max())
    assert np.array_equal(G, G.conj().T)                    # exactly Hermitian, real diagonal
    rng = np.random.default_rng(6)
    S = _lowrank(rng, 30, 40, 6)
    res = orc.greedy(S, np.ones(30), 0.0, 30)
    sigma, kr, X, _ = orc.reconstruct(res, tau2=0.5 ** 3.5)  # sigma_i = 0.5^i
    assert kr == 4 and X.shape == (4, 30)


# ------------------------------------------------------------------------------ GPU parity

@pytest.mark.gpu
@pytest.mark.parametrize("case", ["chirp", "lowrank_real", "lowrank_cplx", "lowrank_real_odd_M"])
def test_gpu_reconstruct_parity(orc, case):
    """(the odd-M real case has an R row pitch that is not a multiple of 16 bytes: the Gram
    kernel's tensor map then reads a padded copy)"""
    from paper_1805_06124_b200 import inputs, rbg
    rng = np.random.default_rng(9)
    if case == "chirp":
        S, w, tol, k_max = inputs.config1(M=6000, N=1000)
        k_max = 60
    else:
        S = _lowrank(rng, 300, 4999 if case.endswith("odd_M") else 5000, 40, case == "lowrank_cplx", decay=0.8)
        w = rng.uniform(0.5, 1.5, 300)
        tol, k_max = 0.0, 300
    res = orc.greedy(S, w, tol, k_max)
    s_o, kr_o, X_o, _ = orc.reconstruct(res, 1e-3)
    with rbg.Context(S, w, tol, k_max) as ctx:
        ctx.run()
        G = ctx.gram()
        s_g, kr_g, X_g = ctx.reconstruct(1e-3)
    np.testing.assert_array_equal(G, orc.gram(res.R))          # same order: bit for bit
    np.testing.assert_allclose(s_g, s_o, rtol=0, atol=1e-12 * s_o[0])
    assert kr_g == kr_o
    # columns agree up to a unit phase where the singular value is separated
    gaps = np.abs(np.diff(s_o))
    for j in range(kr_o):
        sep = min(gaps[j - 1] if j else np.inf, gaps[j] if j < len(gaps) else np.inf)
        if sep < 1e-6 * s_o[0]:
            continue
        ph = np.vdot(X_o[j] * w, X_g[j])
        assert abs(abs(ph) - 1) < 1e-8
        np.testing.assert_allclose(X_g[j], ph * X_o[j], atol=1e-8 * np.abs(X_o[j]).max())
    # the GPU basis is W-orthonormal
    Gx = (X_g.conj() * w) @ X_g.T
    np.testing.assert_allclose(Gx, np.eye(kr_g), atol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("split", [(0, 8192, 12388), (0, 4096, 8192, 12388), (0, 5000, 12388)])
def test_gpu_sharded_gram_fold_and_reconstruct(orc, split):
    """Sharded Algorithm 4 (rbg_gram_fold + rbg_reconstruct_gram, R33): column-sharded
    contexts (EXTERNAL exchange, one GPU) fold the Gram matrix in rank order.  Chunk-aligned
    rank blocks reproduce the one-context Gram, singular values and basis bit for bit; an
    unaligned split gives the oracle's per-rank chunked fold bit for bit and the one-context
    Gram to rounding."""
    from paper_1805_06124_b200 import inputs, rbg
    S, w, tol, _ = inputs.config1(M=split[-1], N=600)
    k_max = 40
    M = S.shape[0]
    with rbg.Context(S, w, tol, k_max) as ctx1:
        ctx1.run()
        G1 = ctx1.gram()
        s1, kr1, X1 = ctx1.reconstruct(1e-3)
        R1 = ctx1.R()
    world = len(split) - 1
    ctxs = [rbg.Context(S[split[p]:split[p + 1]], w, tol, k_max, comm=rbg.COMM_EXTERNAL, rank=p, world=world,
                        col_offset=split[p], M_global=M) for p in range(world)]
    for _ in range(k_max + 1):
        for c in ctxs:
            c.iter_local()
        rbg.emulate_allgather(ctxs)
        for c in ctxs:
            c.iter_finish()
    G = None
    for c in ctxs:
        G = c.gram_fold(G)
    # the oracle's fold: each rank's 4,096-column chunks of its own block, added in order
    ref = np.zeros_like(G1)
    for p in range(world):
        Rp = R1[:, split[p]:split[p + 1]]
        for j0 in range(0, Rp.shape[1], orc.GRAM_CHUNK):
            ref = ref + orc.gram(Rp[:, j0:j0 + orc.GRAM_CHUNK])
    np.fill_diagonal(ref, ref.diagonal().real)
    np.testing.assert_array_equal(G, ref)
    aligned = all(o % orc.GRAM_CHUNK == 0 for o in split[:-1])
    if aligned:
        np.testing.assert_array_equal(G, G1)
    else:
        np.testing.assert_allclose(G, G1, rtol=0, atol=1e-13 * np.abs(G1).max())
    for c in ctxs:
        s, kr, X = c.reconstruct_gram(G, 1e-3)
        assert kr == kr1
        if aligned:
            np.testing.assert_array_equal(s, s1)
            np.testing.assert_array_equal(X, X1)
        else:
            np.testing.assert_allclose(s, s1, rtol=0, atol=1e-12 * s1[0])
        c.close()
