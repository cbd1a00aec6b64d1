"""Input recipe checks: quadrature exactness, normalisation, shapes."""
import numpy as np

from paper_1805_06124_b200 import inputs


def test_simpson_weights_integrate_cubics_exactly():
    N = 64
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    a, b = -1.0, -1.0 / N                    # the grid's span: Simpson on [t0, t_{N-2}], trapezoid after
    # Simpson part is exact for cubics; the trapezoid interval is exact for linear functions.
    for p in range(2):
        got = np.sum(w * t ** p)
        exact = (b ** (p + 1) - a ** (p + 1)) / (p + 1)
        assert abs(got - exact) < 1e-14
    ws = w.copy()
    h = 1.0 / N
    ws[N - 2] -= h / 2
    ws[N - 1] -= h / 2
    for p in range(4):
        got = np.sum(ws * t ** p)
        bb = t[N - 2]
        exact = (bb ** (p + 1) - a ** (p + 1)) / (p + 1)
        assert abs(got - exact) < 1e-13


def test_chirp_columns_are_w_normalised():
    S, w, tol, k_max = inputs.config1(M=50, N=200)
    assert S.shape == (50, 200) and S.dtype == np.complex128
    np.testing.assert_allclose(np.sum(w[None, :] * np.abs(S) ** 2, axis=1), 1.0, rtol=1e-13)
    S2, w2, tol2, k2 = inputs.config2(M=20, N=200)
    np.testing.assert_allclose(np.sum(w2[None, :] * np.abs(S2) ** 2, axis=1), 1.0, rtol=1e-13)
    assert (tol, k_max, tol2, k2) == (1e-12, 50, 0.0, 20)


def test_configs_are_seeded():
    a = inputs.config0()[0]
    b = inputs.config0()[0]
    np.testing.assert_array_equal(a, b)
    assert a.shape == (512, 256)
    S, w, tol, k_max, (U, sig, V) = inputs.config4(M=256, N=128, r=32)
    assert S.shape == (256, 128) and k_max == 32
    np.testing.assert_allclose(U.T @ U, np.eye(32), atol=1e-13)
    np.testing.assert_allclose(S.T, (U * sig) @ V.T, atol=1e-14)
