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


@pytest.mark.parametrize("mode", ["canonical", "plain"])
def test_oracle_resume_branch_cor56_on_enlarged_set(orc, mode):
    """The oracle's resume branch (rbg_oracle.c, k0 >= 0: enrichment, reading
    R32) pinned directly, in both lane modes.  After every enrichment round, for every k from the
    resume point k0 to the new stop:
      * Cor. 5.6 on the ENLARGED column set: err_k = max_j of the direct
        projection residual ||(I - P_k) s~_j||, computed by explicit projection (brute.py), within
        the recurrence floor (reading R8);
      * the pivot taken at k maximises that direct residual up to the same floor;
      * err is non-increasing from k0 on (slack = the floor)."""
    L = orc.CANONICAL if mode == "canonical" else orc.PLAIN
    S, V, w = _sets(M_train=60)
    tol = 1e-5
    res = orc.greedy(S, w, tol, 150, lanes=L)
    scale = np.sqrt(np.max(np.sum(w * np.abs(np.concatenate([S, V])) ** 2, axis=1)))
    atol = 1e-7 * scale                                  # recurrence floor (R8), as above
    added = np.zeros(V.shape[0], bool)
    rounds = 0
    for _ in range(4):
        err, _, _ = orc.validate(res.Q, V, w, L[0])
        fail = (err >= tol) & ~added
        if not fail.any():
            break
        added |= fail
        _, C, e2 = orc.validate(res.Q, V[fail], w, L[0])
        S = np.concatenate([S, V[fail]])
        res.R = np.concatenate([res.R, C], axis=1)
        res.r2 = np.concatenate([res.r2, e2])
        k0, piv0 = res.k, res.pivots.copy()
        res = orc.greedy(S, w, tol, 150, lanes=L, resume=res)
        rounds += 1
        assert res.k > k0 and np.array_equal(res.pivots[:k0], piv0)     # continued, not restarted
        St = brute.weighted(S, w)
        Qt = brute.weighted(res.Q, w)                    # W^{1/2} q_i: orthonormal in l2
        for k in range(k0, res.k + 1):
            d = brute.direct_residuals(St, Qt[:, :k])
            assert abs(res.errors[k] - d.max()) <= atol, (k, res.errors[k], d.max())
            if k < res.k:
                assert d[res.pivots[k]] >= d.max() - atol
        assert np.all(np.diff(res.errors[k0:]) <= atol)
        assert len(set(res.pivots.tolist())) == res.k    # a permutation prefix (R10)
    assert rounds >= 1


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


@pytest.mark.gpu
def test_gpu_running_greedy_refuses_r_readers(orc):
    """Between rbg_step calls the sweep with q_{k-1} is still pending (R row k-1 not filled):
    add_columns, gram and reconstruct return ESTATE; validate and EIM (basis only) work; after
    the stop decision all of them do."""
    from paper_1805_06124_b200 import rbg
    S, V, w = _sets(M_train=60)
    with rbg.Context(S, w, 0.0, 40) as ctx:
        ctx.step(5)
        assert ctx.info()[::2] == (5, "NONE")
        for call in (lambda: ctx.add_columns(V[:3]), ctx.gram, ctx.reconstruct):
            with pytest.raises(rbg.RbgError) as e:
                call()
            assert e.value.status == rbg.ESTATE
        assert ctx.validate(V).shape == (V.shape[0],)
        assert len(ctx.eim()[0]) == 5
        ctx.run()
        k = ctx.info()[0]
        assert k >= 5 and ctx.gram().shape == (k, k)
        ctx.add_columns(V[:3])
        ctx.gram()                                   # settled: the new columns have all rows


@pytest.mark.gpu
def test_gpu_enrichment_device_v_borrowed_s_not_copied(orc):
    """Enrichment with a device validation set and a borrowed device S: the
    appended columns go to a second, library-owned segment that the sweep streams after the
    caller's columns -- S is never copied (device memory grows by the appended columns and the
    longer R rows only) -- and the run equals the oracle's enrichment bit for bit."""
    import torch

    from paper_1805_06124_b200 import rbg
    S, V, w = _sets(M_train=60)
    tol = 1e-5
    res, _, hist_o, ok_o = orc.enrich(S, V, w, tol, 150, rounds=4)
    St = torch.as_tensor(S, device="cuda")
    Vt = torch.as_tensor(V, device="cuda")
    with rbg.Context(St, w, tol, 150) as ctx:
        ctx.run()
        hist, ok = rbg.enrich(ctx, Vt, tol, rounds=4)
        g = ctx.result()
        G = ctx.gram()                       # R now has a row stride with slack (ldr > M)
    assert ok == ok_o and hist == hist_o
    np.testing.assert_array_equal(G, orc.gram(res.R))
    assert (g.k, g.stop) == (res.k, res.stop)
    for key in ("pivots", "errors", "nu", "Q", "R", "r2"):
        np.testing.assert_array_equal(getattr(g, key), getattr(res, key))
    # memory: a 1.3 GB borrowed S, 64 appended columns
    N, M = 2000, 40960
    big, wb, _, _ = inputs.config1(M=M, N=N)
    Bt = torch.as_tensor(big, device="cuda")
    F = Bt[:64].clone() * (1.0 + 1e-3)
    with rbg.Context(Bt, wb, 0.0, 20) as ctx:
        ctx.run()
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        ctx.add_columns(F)
        free1 = torch.cuda.mem_get_info()[0]
        ctx.run()
        assert ctx.info()[0] == 20 and ctx.R().shape == (20, M + 64)
    assert free0 - free1 < 0.1 * Bt.numel() * 16, (free0 - free1) / 1e9


def _drive(rbg, ctxs, mode, n):
    for _ in range(n):
        for c in ctxs:
            c.iter_local()
        if mode == "external":
            rbg.emulate_allgather(ctxs)
        for c in ctxs:
            c.iter_finish()


@pytest.mark.gpu
@pytest.mark.parametrize("mode,cplx", [("peer", True), ("external", True), ("peer", False)])
def test_gpu_sharded_enrichment_bit_exact(orc, mode, cplx):
    """Enrichment of a 2-rank column-sharded greedy (rbg_add_columns_ex, R34): each
    rank validates its own block of V and appends its failing columns with global ids numbered
    in rank order (dist.enrich_plan); the pivot search restarts on every rank with a new record
    epoch.  Pivots, errors, Q, the history and R / r2 (gathered by global column id) equal the
    single-process oracle enrichment of the concatenated V bit for bit."""
    import torch

    from paper_1805_06124_b200 import dist as D
    from paper_1805_06124_b200 import rbg
    S, V, w = _sets(M_train=60)
    if not cplx:
        S, V = S.real.copy(), V.real.copy()
    tol, k_max, rounds = 1e-5, 150, 4
    res, S2, hist_o, ok_o = orc.enrich(S, V, w, tol, k_max, rounds=rounds)
    M, Mv = S.shape[0], V.shape[0]
    sb, vb = [0, 23, M], [0, Mv // 3, Mv]            # ranks' training / validation blocks
    comm = rbg.COMM_PEER if mode == "peer" else rbg.COMM_EXTERNAL
    stream = torch.cuda.Stream()
    ctxs = [rbg.Context(S[sb[p]:sb[p + 1]], w, tol, k_max, stream=stream.cuda_stream, comm=comm, rank=p, world=2,
                        col_offset=sb[p], M_global=M) for p in range(2)]
    if mode == "peer":
        rbg.peer_connect_local(ctxs)
    gids = [list(range(sb[p], sb[p + 1])) for p in range(2)]
    _drive(rbg, ctxs, mode, k_max + 1)
    Vb = [V[vb[p]:vb[p + 1]] for p in range(2)]
    added = [np.zeros(vb[p + 1] - vb[p], bool) for p in range(2)]
    total, hist, ok = M, [], None
    for _ in range(rounds):
        errs = [ctxs[p].validate(Vb[p]) for p in range(2)]
        hist.append(max(float(e.max()) for e in errs))
        fails = [(errs[p] >= tol) & ~added[p] for p in range(2)]
        counts = [int(f.sum()) for f in fails]
        if sum(counts) == 0:
            ok = all(bool(np.all(e < tol)) for e in errs)
            break
        for p in range(2):
            first, total_new = D.enrich_plan(counts, p, total)
            ctxs[p].add_columns(Vb[p][fails[p]], first_gid=first, M_global=total_new)
            gids[p] += list(range(first, first + counts[p]))
            added[p] |= fails[p]
        total = total_new
        _drive(rbg, ctxs, mode, k_max + 1)
    if ok is None:
        errs = [ctxs[p].validate(Vb[p]) for p in range(2)]
        hist.append(max(float(e.max()) for e in errs))
        ok = all(bool(np.all(e < tol)) for e in errs)
    assert ok == ok_o and hist == hist_o
    out = [c.result() for c in ctxs]
    for g in out:
        assert (g.k, g.stop) == (res.k, res.stop)
        np.testing.assert_array_equal(g.pivots, res.pivots)
        np.testing.assert_array_equal(g.errors, res.errors)
        np.testing.assert_array_equal(g.Q, res.Q)
    R = np.zeros_like(res.R)
    r2 = np.zeros_like(res.r2)
    for p in range(2):
        R[:, gids[p]] = out[p].R
        r2[gids[p]] = out[p].r2
    np.testing.assert_array_equal(R, res.R)
    np.testing.assert_array_equal(r2, res.r2)
    for c in ctxs:
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("cplx,N,M_v,k", [
    (True, 400, 37, 35),      # ragged column and basis tiles, 6.25 stages of 64 rows
    (True, 400, 16, 16),      # exactly one tile
    (True, 400, 5, 1),        # one basis vector
    (False, 257, 50, 33),     # real, odd N (padding row in the last 16-byte vector)
    (False, 128, 17, 20),     # real, N a multiple of the stage
    (True, 2000, 1000, 100),  # config-1 rows, many CTAs per column tile
])
def test_gpu_coefficient_block_bit_exact(orc, monkeypatch, cplx, N, M_v, k):
    """The blocked coefficient kernel (coeff.cu: all k basis vectors in one pass over V) gives
    the oracle's errors and coefficients bit for bit, and the same bits as the k streaming
    coefficient sweeps it replaces (RBG_COEFF=passes), across tile edges and ragged tails."""
    from paper_1805_06124_b200 import rbg
    if N % 2:   # odd N (Simpson needs even N): Gaussian columns, weights U[0.5, 1.5]
        rng = np.random.default_rng(7)
        S, V = rng.standard_normal((max(2 * k, 60), N)), rng.standard_normal((M_v, N))
        w = rng.uniform(0.5, 1.5, N)
    else:
        S, w, _, _ = inputs.config1(M=max(2 * k, 60), N=N)
        t = inputs.chirp_grid(N)
        q, chi, psi = inputs.chirp_params(M_v, 13, spin=False)
        V = inputs.chirp_columns(t, w, q, chi, psi, spin=False)
    if not cplx:
        S, V = S.real.copy(), V.real.copy()
    r = orc.greedy(S, w, 0.0, k)
    assert r.k == k or r.k > 16              # RANK may stop early; still several basis tiles
    e_o, C_o, _ = orc.validate(r.Q, V, w)
    with rbg.Context(S, w, 0.0, k) as ctx:
        ctx.run()
        err, C = ctx.validate(V, coeffs=True)
        monkeypatch.setenv("RBG_COEFF", "passes")
        err_p, C_p = ctx.validate(V, coeffs=True)
    np.testing.assert_array_equal(err, e_o)
    np.testing.assert_array_equal(C, C_o)
    np.testing.assert_array_equal(err_p, err)
    np.testing.assert_array_equal(C_p, C)


@pytest.mark.gpu
@pytest.mark.parametrize("cplx,N,pad", [
    (True, 400, 0),     # complex: column pitch = the padded layout -> read in place
    (False, 256, 0),    # real, N even -> read in place
    (False, 257, 0),    # real, N odd: the padded layout has one more row -> copied
    (True, 400, 3),     # row stride N + 3 -> copied
])
def test_gpu_validate_device_blocks(orc, cplx, N, pad):
    """A CUDA-tensor block is validated in place when its layout is the library's padded one
    and copied otherwise; both give the oracle's bits, and a non-finite entry of a device
    block is reported (ENONFINITE) in either case."""
    import torch

    from paper_1805_06124_b200 import rbg
    rng = np.random.default_rng(N + pad)
    S = rng.standard_normal((80, N)) + (1j * rng.standard_normal((80, N)) if cplx else 0)
    V = rng.standard_normal((45, N)) + (1j * rng.standard_normal((45, N)) if cplx else 0)
    w = rng.uniform(0.5, 1.5, N)
    r = orc.greedy(S, w, 0.0, 30)
    e_o, C_o, _ = orc.validate(r.Q, V, w)
    dt = torch.complex128 if cplx else torch.float64
    buf = torch.zeros((45, N + pad), dtype=dt, device="cuda")
    buf[:, :N] = torch.from_numpy(V).to("cuda")
    Vd = buf[:, :N]
    with rbg.Context(S, w, 0.0, 30) as ctx:
        ctx.run()
        err, C = ctx.validate(Vd, coeffs=True)
        np.testing.assert_array_equal(err, e_o)
        np.testing.assert_array_equal(C, C_o)
        buf[7, 3] = float("nan")
        with pytest.raises(rbg.RbgError, match="ENONFINITE"):
            ctx.validate(Vd)
