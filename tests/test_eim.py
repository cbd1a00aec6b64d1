"""Empirical interpolation nodes (DESIGN.md NEXT f-2, reading R31).

Oracle pins: SPEC.md's closed forms (identity basis, a single vector), exact reproduction of
span(Q) from node samples, distinct nodes, the DEIM error bound
||u - I[u]||_2 <= ||B^{-1}||_2 ||(I - Q Q^H) u||_2 (orthonormal Q, Chaturantabut-Sorensen),
and the interpolation of training snapshots.  GPU parity: nodes and B bit for bit.
"""
import numpy as np
import pytest

from paper_1805_06124_b200 import inputs


def test_closed_forms(orc):
    nodes, B = orc.eim(np.eye(5)[:3])          # Q = first 3 unit vectors in R^5
    assert list(nodes) == [0, 1, 2]
    np.testing.assert_array_equal(B, np.eye(3))
    nodes, B = orc.eim(np.array([[0.6, 0.8]]))
    assert list(nodes) == [1] and B[0, 0] == 0.8
    # exact tie between rows 2 and 5 of the first vector: lowest row
    q = np.zeros((1, 7))
    q[0, 2] = q[0, 5] = -1.0
    assert list(orc.eim(q)[0]) == [2]


@pytest.mark.parametrize("cplx", [True, False])
def test_span_reproduction_and_deim_bound(orc, cplx):
    S, w, _, _ = inputs.config1(M=400, N=300)
    if not cplx:
        S = S.real.copy()
    w1 = np.ones(S.shape[1])                     # unweighted: Q orthonormal in l2
    res = orc.greedy(S, w1, 0.0, 40)
    Q = res.Q
    nodes, B = orc.eim(Q)
    k = res.k
    assert len(set(nodes.tolist())) == k
    np.testing.assert_array_equal(B, Q[:, nodes].T)
    # q_j is reproduced from its samples
    for j in (0, 7, k - 1):
        c = np.linalg.solve(B, Q[j, nodes])
        np.testing.assert_allclose(Q.T @ c, Q[j], atol=1e-10)
    # DEIM bound on training snapshots
    Binv = np.linalg.norm(np.linalg.inv(B), 2)
    for s in S[::37]:
        interp = Q.T @ np.linalg.solve(B, s[nodes])
        proj = s - Q.T @ (Q.conj() @ s)
        assert np.linalg.norm(s - interp) <= Binv * np.linalg.norm(proj) * (1 + 1e-8) + 1e-12


def test_degenerate_basis(orc):
    Q = np.array([[1.0, 0.0, 0.0], [2.0, 0.0, 0.0]])   # second vector in span of the first
    assert orc.eim(Q) is None


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg1", "cfg4", "cfg0", "cfg4_k336", "gauss_k600"])
def test_gpu_eim_bit_exact(orc, monkeypatch, case):
    """GPU EIM nodes and node matrix equal the oracle's bit for bit, for the warp-level
    forward substitution (1..32 register slots per lane: k up to 600 here) and for the first
    block-barrier version (RBG_EIM=block)."""
    from paper_1805_06124_b200 import rbg
    if case == "cfg1":
        S, w, tol, k_max = inputs.config1(M=3000, N=2000)
        k_max = 120
    elif case == "cfg4":
        S, w, tol, k_max, _ = inputs.config4(M=4096, N=1024, r=256)
    elif case == "cfg4_k336":
        S, w, tol, k_max, _ = inputs.config4(M=2048, N=1024, r=400)   # RANK stop at k = 336
    elif case == "gauss_k600":
        rng = np.random.default_rng(600)
        S, w, tol, k_max = rng.standard_normal((700, 1031)), rng.uniform(0.5, 1.5, 1031), 0.0, 600
    else:
        S, w, tol, k_max = inputs.config0()
    res = orc.greedy(S, w, tol, k_max)
    nodes_o, B_o = orc.eim(res.Q)
    with rbg.Context(S, w, tol, k_max) as ctx:
        ctx.run()
        nodes, B = ctx.eim()
        monkeypatch.setenv("RBG_EIM", "block")
        nodes1, B1 = ctx.eim()
    np.testing.assert_array_equal(nodes, nodes_o)
    np.testing.assert_array_equal(B, B_o)
    np.testing.assert_array_equal(nodes1, nodes_o)
    np.testing.assert_array_equal(B1, B_o)
