"""Out-of-sample validation and enrichment (DESIGN.md NEXT f-1).

Oracle pins (CPU) and GPU parity (marked gpu).  The validation error of a column is the
greedy's own projection error ||v - Q Q^H W v||_w evaluated with the residual recurrence;
enrichment appends failing validation columns to the training set and continues the greedy.
"""
import numpy as np
import pytest

import brute
from paper_1805_06124_b200 import inputs


def _sets(M_train=150, M_val=300, N=400):
    S, w, _, _ = inputs.config1(M=M_train, N=N)
    t = inputs.chirp_grid(N)
    q, chi, psi = inputs.chirp_params(M_val, 11, spin=False)   # independent parameter draw
    V = inputs.chirp_columns(t, w, q, chi, psi, spin=False)
    return S, V, w


# ------------------------------------------------------------------------------ oracle pins

def test_training_set_passes_at_training_tolerance(orc):
    """Cor. 5.6: after a TOL stop every training column has error < tol."""
    S, V, w = _sets()
    tol = 1e-6
    r = orc.greedy(S, w, tol, 150)
    assert r.stop == "TOL"
    err, C, e2 = orc.validate(r.Q, S, w)
    assert np.all(err < tol)
    # and the validation residual of an unselected training column IS the greedy's residual
    unsel = np.setdiff1d(np.arange(S.shape[0]), r.pivots)
    np.testing.assert_array_equal(e2[unsel], r.r2[unsel])
    np.testing.assert_array_equal(C, r.R)


def test_validation_matches_direct_projection(orc):
    S, V, w = _sets()
    r = orc.greedy(S, w, 0.0, 40)
    err, C, _ = orc.validate(r.Q, V, w)
    Qt = (np.sqrt(w)[None, :] * r.Q).T
    Vt = brute.weighted(V, w)
    d = brute.direct_residuals(Vt, Qt)
    scale = np.sqrt(np.max(np.sum(w * np.abs(V) ** 2, axis=1)))
    np.testing.assert_allclose(err, d, atol=1e-7 * scale)          # recurrence floor (R8)
    np.testing.assert_allclose(C, (r.Q.conj() * w) @ V.T, atol=1e-13)


def test_orthogonal_unit_vector_has_error_one(orc):
    """a vector W-orthogonal to span(Q) with ||.||_w = 1 has error 1."""
    N = 16
    w = np.full(N, 0.25)
    Q = np.zeros((3, N))
    Q[0, 0] = Q[1, 1] = Q[2, 2] = 2.0                  # W-orthonormal (w q^2 = 1)
    v = np.zeros((1, N))
    v[0, 5] = 2.0
    err, C, _ = orc.validate(Q, v, w)
    assert err[0] == 1.0 and np.all(C == 0)
    err, _, _ = orc.validate(np.zeros((0, N)), v, w)   # empty basis: the norm
    assert err[0] == 1.0


def test_enrichment_converges_and_is_monotone(orc):
    S, V, w = _sets(M_train=60)
    tol = 1e-5
    res, S2, hist, ok = orc.enrich(S, V, w, tol, 150, rounds=4)
    assert len(hist) >= 2 and hist[0] >= tol           # validation failed at first
    assert ok and res.stop == "TOL"
    assert all(b <= a for a, b in zip(hist, hist[1:]))  # non-increasing
    # the continued greedy equals a greedy over the enlarged set that is forced to reuse the
    # first basis: every training column (incl. appended ones) is now below tol
    err, _, _ = orc.validate(res.Q, S2, w)
    assert np.all(err < tol)
    G = (res.Q.conj() * w) @ res.Q.T
    assert np.max(np.abs(G - np.eye(res.k))) <= 1e-12


# ------------------------------------------------------------------------------ GPU parity

@pytest.mark.gpu
def test_gpu_validate_bit_exact(orc):
    from paper_1805_06124_b200 import rbg
    S, V, w = _sets()
    r = orc.greedy(S, w, 0.0, 60)
    with rbg.Context(S, w, 0.0, 60) as ctx:
        ctx.run()
        err, C = ctx.validate(V, coeffs=True)
        err0 = ctx.validate(S[:7])
    e_o, C_o, _ = orc.validate(r.Q, V, w)
    np.testing.assert_array_equal(err, e_o)
    np.testing.assert_array_equal(C, C_o)
    np.testing.assert_array_equal(err0, orc.validate(r.Q, S[:7], w)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("cplx", [True, False])
def test_gpu_enrichment_bit_exact(orc, cplx):
    from paper_1805_06124_b200 import rbg
    S, V, w = _sets(M_train=60)
    if not cplx:
        S, V = S.real.copy(), V.real.copy()
    tol = 1e-5
    res, S2, hist_o, ok_o = orc.enrich(S, V, w, tol, 150, rounds=4)
    with rbg.Context(S, w, tol, 150) as ctx:
        ctx.run()
        hist, ok = rbg.enrich(ctx, V, tol, rounds=4)
        g = ctx.result()
    assert ok == ok_o and hist == hist_o
    assert (g.k, g.stop) == (res.k, res.stop)
    np.testing.assert_array_equal(g.pivots, res.pivots)
    np.testing.assert_array_equal(g.errors, res.errors)
    np.testing.assert_array_equal(g.Q, res.Q)
    np.testing.assert_array_equal(g.R, res.R)
