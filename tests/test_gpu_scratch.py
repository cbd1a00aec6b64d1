"""The NEXT-row calls keep their device work buffers in a per-context scratch pool (DESIGN.md
"Host side of the NEXT-row calls"): a slot is reused, grown when a call needs more, and shared
by calls that never run at the same time (rbg_gram / rbg_gram_fold / rbg_reconstruct).  Reuse
must not change a single bit: every call in a mixed sequence on one context returns what the
oracle (or the same call on a fresh context) returns."""
import numpy as np
import pytest

from paper_1805_06124_b200 import inputs


def _val_block(M, N, seed):
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(M, seed, spin=False)
    return inputs.chirp_columns(t, w, q, chi, psi, spin=False)


@pytest.mark.gpu
def test_gpu_validation_pool_growth_and_shrink(orc):
    """Validation blocks of 40, 500, 40 and 500 columns on one context (the pooled buffers grow,
    are reused larger than needed, and are reused again): errors and coefficients equal the
    oracle's bit for bit every time."""
    from paper_1805_06124_b200 import rbg
    S, w, _, _ = inputs.config1(M=600, N=700)
    res = orc.greedy(S, w, 0.0, 60)
    with rbg.Context(S, w, 0.0, 60) as ctx:
        ctx.run()
        for M_v, seed in ((40, 21), (500, 22), (40, 23), (500, 24)):
            V = _val_block(M_v, 700, seed)
            err, C = ctx.validate(V, coeffs=True)
            err_o, C_o, _ = orc.validate(res.Q, V, w)
            np.testing.assert_array_equal(err, err_o)
            np.testing.assert_array_equal(C, C_o)


@pytest.mark.gpu
def test_gpu_gram_reconstruct_eim_interleaved():
    """gram, reconstruct, gram_fold, EIM and reconstruct again on one context share pooled
    buffers; each repeated call returns exactly what the same call returns on a fresh context."""
    from paper_1805_06124_b200 import rbg
    S, w, _, k_max = inputs.config1(M=2000, N=2000)   # X of 2.9 MB: the page-locked output path
    k_max = 90

    def fresh(what):
        with rbg.Context(S, w, 0.0, k_max) as c:
            c.run()
            return what(c)

    G_ref = fresh(lambda c: c.gram())
    sig_ref, kr_ref, X_ref = fresh(lambda c: c.reconstruct(1e-6))
    nodes_ref, B_ref = fresh(lambda c: c.eim())
    with rbg.Context(S, w, 0.0, k_max) as ctx:
        ctx.run()
        for _ in range(2):
            np.testing.assert_array_equal(ctx.gram(), G_ref)
            sig, kr, X = ctx.reconstruct(1e-6)
            assert kr == kr_ref
            np.testing.assert_array_equal(sig, sig_ref)
            np.testing.assert_array_equal(X, X_ref)
            G2 = ctx.gram_fold(np.zeros_like(G_ref))
            np.testing.assert_array_equal(G2, G_ref)
            nodes, B = ctx.eim()
            np.testing.assert_array_equal(nodes, nodes_ref)
            np.testing.assert_array_equal(B, B_ref)
