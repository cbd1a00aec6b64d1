"""Golden closed-form cases (tests/golden/closed_forms.json, each with the passage that fixes
it): the CPU oracle (CPU tests) and the CUDA path through the C ABI (GPU tests) must reproduce
them.  These are values written down from the paper / SPEC by hand, not produced by running
either implementation."""
import json
import os

import numpy as np
import pytest

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def _case(c):
    S = np.array(c["S"], dtype=np.float64)
    w = np.array(c["w"], dtype=np.float64) if "w" in c else np.ones(S.shape[1])
    return S, w, float(c["tol"]), int(c["k_max"])


def _check(c, k, stop, pivots, errors):
    assert stop == c["stop"], (c["name"], stop)
    assert list(pivots) == c["pivots"], (c["name"], list(pivots))
    assert k == len(c["pivots"])
    exp = np.array(c["errors"], dtype=np.float64)
    got = np.asarray(errors)[:len(exp)] if c.get("errors_prefix") else np.asarray(errors)
    np.testing.assert_allclose(got, exp, rtol=1e-15, atol=0, err_msg=c["cite"])


@pytest.mark.parametrize("c", GOLDEN["greedy"], ids=[c["name"] for c in GOLDEN["greedy"]])
@pytest.mark.parametrize("lanes", ["canonical", "plain"])
def test_oracle_golden_greedy(orc, c, lanes):
    S, w, tol, k_max = _case(c)
    r = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL if lanes == "canonical" else orc.PLAIN)
    _check(c, r.k, r.stop, r.pivots, r.errors)


@pytest.mark.parametrize("c", GOLDEN["imgs"], ids=[c["name"] for c in GOLDEN["imgs"]])
def test_oracle_golden_imgs(orc, c):
    v = np.array(c["v"], dtype=np.float64)
    Q = np.array(c["Q"], dtype=np.float64).reshape(-1, v.shape[0])
    out = orc.imgs(Q, v, np.ones(v.shape[0]), orc.CANONICAL[1])
    assert out is not None, c["cite"]
    q, coeff, _, nu = out
    np.testing.assert_allclose(q, c["q"], atol=1e-14, err_msg=c["cite"])
    if "coeffs" in c:
        np.testing.assert_allclose(coeff, c["coeffs"], atol=1e-14, err_msg=c["cite"])
    assert nu == c["nu"]


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLDEN["greedy"], ids=[c["name"] for c in GOLDEN["greedy"]])
def test_gpu_golden_greedy(c):
    from paper_1805_06124_b200 import rbg
    S, w, tol, k_max = _case(c)
    g = rbg.greedy(S, w, tol, k_max)
    _check(c, g.k, g.stop, g.pivots, g.errors)
