"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, same seeded inputs.

Canonical mode (lanes (32, 2048)) evaluates the same floating-point expression DAG as
the kernels, so pivots, stop reason, k, nu
are compared exactly and Q, R, errors, r2 bit for bit.  BASELINE.json's tolerance
(1e-10 relative) is asserted as well so that a failure says which bar was missed.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1805_06124_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rbg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1805_06124_b200 import build as B
    B.build()
    from paper_1805_06124_b200 import rbg as R
    return R


def compare(g, o, scale=None, exact=True):
    """g: rbg.Result, o: oracle.GreedyResult."""
    assert (g.k, g.stop) == (o.k, o.stop), ((g.k, g.stop), (o.k, o.stop))
    np.testing.assert_array_equal(g.pivots, o.pivots)
    np.testing.assert_array_equal(g.nu, o.nu)
    # BASELINE.json bar: 1e-10 relative (per column for R)
    s = scale if scale is not None else max(o.errors[0], 1e-300)
    np.testing.assert_allclose(g.errors, o.errors, rtol=0, atol=1e-10 * s)
    np.testing.assert_allclose(g.Q, o.Q, rtol=0, atol=1e-10 * np.abs(o.Q).max(initial=1.0))
    np.testing.assert_allclose(g.R, o.R, rtol=0, atol=1e-10 * s)
    if exact:  # the canonical contract: 0 ulp
        np.testing.assert_array_equal(g.errors, o.errors)
        np.testing.assert_array_equal(g.rdiag, o.rdiag)
        np.testing.assert_array_equal(g.Q, o.Q)
        np.testing.assert_array_equal(g.R, o.R)
        np.testing.assert_array_equal(g.r2, o.r2)


def both(rbg, orc, S, w, tol, k_max, **kw):
    g = rbg.greedy(S, w, tol, k_max, **kw)
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    return g, o


def test_config0_full(rbg, orc):
    S, w, tol, k_max = inputs.config0()
    g, o = both(rbg, orc, S, w, tol, k_max)
    compare(g, o)
    assert g.stop == "RANK"          # reading R8: the recurrence floor stops it by rank


def test_config1_reduced(rbg, orc):
    S, w, tol, k_max = inputs.config1(M=3000, N=2000)
    g, o = both(rbg, orc, S, w, tol, k_max)
    compare(g, o)


def test_config1_full(rbg, orc):
    S, w, tol, k_max = inputs.config1()
    g, o = both(rbg, orc, S, w, tol, k_max)
    compare(g, o)


def test_config2_reduced(rbg, orc):
    S, w, tol, k_max = inputs.config2(M=3000, N=10000)
    g, o = both(rbg, orc, S, w, tol, 60)
    compare(g, o)
    assert g.stop == "KMAX"


def test_config4_reduced(rbg, orc):
    S, w, tol, k_max, _ = inputs.config4(M=4096, N=1024, r=256)
    g, o = both(rbg, orc, S, w, tol, k_max)
    compare(g, o)


@pytest.mark.parametrize("N,M,cplx", [(1, 1, False), (1, 7, True), (7, 1, True), (33, 5, False),
                                      (257, 1000, False), (255, 3, True), (4097, 300, True),
                                      (2049, 64, False), (100, 2000, True),
                                      # staged IMGS limit, global-memory e~ (N*16 B > smem),
                                      # unstaged IMGS (12/16 vectors per lane), maximum N
                                      (16384, 40, True), (14000, 33, True), (20000, 24, True),
                                      (32768, 20, True), (30001, 25, False), (65536, 12, False)])
def test_ragged_shapes(rbg, orc, N, M, cplx):
    """Odd N (real padding row), N not a multiple of 32 / 2048, M below the grid size,
    single row / single column."""
    rng = np.random.default_rng(N * 7919 + M)
    S = rng.standard_normal((M, N)) + (1j * rng.standard_normal((M, N)) if cplx else 0)
    w = rng.uniform(0.5, 1.5, N)
    k_max = min(N, M, 40)
    g, o = both(rbg, orc, S, w, 0.0, k_max)
    compare(g, o)


@pytest.mark.parametrize("N,cplx", [(128, True), (129, True), (256, True), (257, True), (512, True), (513, True),
                                     (255, False), (257, False), (1023, False), (1025, False), (2048, True),
                                     (2049, True)])
def test_imgs_cluster_size_boundaries(rbg, orc, N, cplx):
    """nvec around the IMGS layout switches (1, 2, 4 CTAs of 128 lanes up to 512 vectors, then the
    16-CTA cluster; one vector per lane up to 2,048): same bits on both sides of each boundary,
    with enough iterations for two MGS passes per pivot and an odd and even basis size."""
    rng = np.random.default_rng(N * 131 + cplx)
    M = 300
    S = rng.standard_normal((M, N)) + (1j * rng.standard_normal((M, N)) if cplx else 0)
    w = rng.uniform(0.5, 1.5, N)
    for k_max in (37, 40):
        g, o = both(rbg, orc, S, w, 0.0, k_max)
        compare(g, o)


def test_degenerate_inputs(rbg, orc):
    g = rbg.greedy(np.zeros((5, 4)), None, 0.0, 3)
    assert (g.k, g.stop, list(g.errors)) == (0, "RANK", [0.0])
    g = rbg.greedy(np.eye(3), None, 0.0, 3)
    assert (g.k, g.stop, list(g.pivots), list(g.errors)) == (3, "ALL_SELECTED", [0, 1, 2], [1, 1, 1, 0])
    g = rbg.greedy(np.diag([3.0, 2.0, 1.0]), None, 1.5, 3)
    assert (g.k, g.stop, list(g.errors)) == (2, "TOL", [3.0, 2.0, 1.0])
    g = rbg.greedy(np.diag([3.0, 2.0, 1.0]), None, 0.0, 2)
    assert (g.k, g.stop) == (2, "KMAX")
    g = rbg.greedy(np.eye(4)[:2], None, 0.0, 3)                  # k_max > M
    assert (g.k, g.stop, list(g.errors)) == (2, "ALL_SELECTED", [1, 1, 0])
    # exact ties: lowest global index
    S = np.ones((6, 4))
    g = rbg.greedy(S, None, 0.0, 2)
    assert g.pivots[0] == 0 and g.stop == "RANK"


def test_device_tensor_borrowed_and_strided(rbg, orc):
    import torch
    S, w, tol, k_max = inputs.config1(M=1500, N=512)
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    St = torch.as_tensor(S, device="cuda")
    g = rbg.greedy(St, torch.as_tensor(w, device="cuda"), tol, k_max)
    compare(g, o)
    big = torch.zeros((1500, 520), dtype=torch.complex128, device="cuda")
    big[:, :512] = St
    g2 = rbg.greedy(big[:, :512], w, tol, k_max)          # ld = 520 > N
    compare(g2, o)
    g3 = rbg.greedy(St, w, tol, k_max, borrow=False)      # device copy path
    compare(g3, o)


def test_nonfinite_input(rbg):
    import torch
    S = torch.ones((10, 8), dtype=torch.float64, device="cuda")
    S[6, 3] = float("nan")
    with pytest.raises(rbg.RbgError) as e:
        rbg.greedy(S, None, 0.0, 3)
    assert e.value.status == rbg.ENONFINITE and "row 3, col 6" in str(e.value)
    H = np.ones((5, 4), np.complex128)
    H[3, 2] = complex(1.0, np.inf)
    with pytest.raises(rbg.RbgError) as e:
        rbg.greedy(H, None, 0.0, 3)
    assert e.value.status == rbg.ENONFINITE and "row 2, col 3" in str(e.value)


def test_graph_batches_match_plain(rbg, orc):
    S, w, tol, k_max = inputs.config1(M=2000, N=1000)
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    with rbg.Context(S, w, tol, k_max) as ctx:
        ctx.set_graph_batch(8)
        ctx.run()
        compare(ctx.result(), o)


@pytest.mark.parametrize("ortho", ["mgs", "cgs"])
def test_device_loop_stops_without_tail(rbg, orc, ortho):
    """rbg_run's device loop (a conditional WHILE graph node over one iteration, the stopping
    kernel clears the condition): the oracle's bits, and no iteration launched past the stop;
    the polled path (timing mode) stops within two batches of 16."""
    S, w, tol, k_max = inputs.config0()
    lanes = orc.CANONICAL_CGS if ortho == "cgs" else orc.CANONICAL
    o = orc.greedy(S, w, tol, k_max, lanes=lanes, ortho=ortho)
    assert o.stop == "RANK" and o.k < k_max - 40       # a tail of > 40 iterations would exist
    loop = not os.environ.get("RBG_NO_DEVICE_LOOP")   # the A/B switch selects the polled path
    with rbg.Context(S, w, tol, k_max, ortho=ortho) as ctx:
        ctx.run()
        compare(ctx.result(), o)
        n0 = ctx.stats().noop_iters
        assert n0 == 0 or not loop
        ctx.run()                                      # already stopped: nothing launched
        assert ctx.stats().noop_iters == n0
    with rbg.Context(S, w, tol, k_max, ortho=ortho) as ctx:
        ctx.set_timing(True)
        ctx.run()
        compare(ctx.result(), o)
        assert 0 <= ctx.stats().noop_iters <= 32


def test_step_api_and_timing_identity(rbg):
    """rbg_step enqueues iterations; the cost-model identity T = T_sweep + T_xchg + T_IMGS
     holds to 1% from the library's own events."""
    S, w, tol, k_max = inputs.config2(M=20000, N=4000)
    with rbg.Context(S, w, tol, 40) as ctx:
        ctx.step(10)
        k, _, why = ctx.info()
        assert (k, why) == (10, "NONE")
        ctx.step(3)
        ctx.run()
        assert ctx.info()[::2] == (40, "KMAX")
    with rbg.Context(S, w, tol, 40) as ctx:
        ctx.set_timing(True)
        ctx.step(10)                  # no host synchronisation between step and run
        ctx.run()
        st = ctx.stats()
        assert st.k == 40 and st.sweeps == 40
        # C_j = exchange + launch gaps between iterations
        c_j = st.t_xchg_ms + st.t_gap_ms
        parts = st.t_init_ms + st.t_sweep_ms + c_j + st.t_imgs_ms
        assert abs(st.t_total_ms - parts) <= 0.01 * st.t_total_ms
        assert st.t_gap_ms <= 0.05 * st.t_total_ms
        sw, xc, im = ctx.timings(40)
        assert np.all(np.isfinite(sw)) and np.all(sw > 0)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_path_on_one_gpu(rbg, orc, world):
    """The column-sharded algorithm (EXTERNAL exchange) gives the single-GPU results bit
    for bit: per-column arithmetic is partition independent and the maxloc order total."""
    S, w, tol, k_max = inputs.config1(M=3001, N=700)
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    M = S.shape[0]
    bounds = [M * p // world for p in range(world + 1)]
    ctxs = [rbg.Context(S[bounds[p]:bounds[p + 1]], w, tol, k_max, comm=rbg.COMM_EXTERNAL,
                        rank=p, world=world, col_offset=bounds[p], M_global=M)
            for p in range(world)]
    for _ in range(k_max + 1):
        for c in ctxs:
            c.iter_local()
        rbg.emulate_allgather(ctxs)
        for c in ctxs:
            c.iter_finish()
    res = [c.result() for c in ctxs]
    for r in res:
        assert (r.k, r.stop) == (o.k, o.stop)
        np.testing.assert_array_equal(r.pivots, o.pivots)
        np.testing.assert_array_equal(r.errors, o.errors)
        np.testing.assert_array_equal(r.Q, o.Q)
    R = np.concatenate([r.R for r in res], axis=1)
    np.testing.assert_array_equal(R, o.R)
    np.testing.assert_array_equal(np.concatenate([r.r2 for r in res]), o.r2)
    for c in ctxs:
        c.close()


def test_nccl_exchange_path_world1(rbg, orc):
    """comm = NCCL with one rank runs the whole exchange path on one GPU: libnccl loaded at
    run time, ncclCommInitRank, the sweep's candidate-column pack, ncclAllGather on the
    library stream and the decision from the gathered records -- bit-identical results."""
    S, w, tol, k_max = inputs.config1(M=2500, N=800)
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    uid = rbg.unique_id()
    assert len(uid) == 128
    with rbg.Context(S, w, tol, k_max, comm=rbg.COMM_NCCL, rank=0, world=1, nccl_id=uid) as ctx:
        ctx.set_timing(True)
        ctx.run()
        compare(ctx.result(), o)
        st = ctx.stats()
        assert st.t_xchg_ms > 0.0
    with rbg.Context(S, w, tol, k_max, comm=rbg.COMM_EXTERNAL, rank=0, world=1) as ctx:
        for _ in range(k_max + 1):
            ctx.iter_local()
            rbg.emulate_allgather([ctx])
            ctx.iter_finish()
        compare(ctx.result(), o)


def _peer_group(rbg, S, w, tol, k_max, world, stream, **kw):
    M = S.shape[0]
    bounds = [M * p // world for p in range(world + 1)]
    ctxs = [rbg.Context(S[bounds[p]:bounds[p + 1]], w, tol, k_max, stream=stream, comm=rbg.COMM_PEER,
                        rank=p, world=world, col_offset=bounds[p], M_global=M, peer_timeout_ms=20000, **kw)
            for p in range(world)]
    if world > 1:
        rbg.peer_connect_local(ctxs)
    return ctxs


@pytest.mark.parametrize("world,ortho", [(1, "mgs"), (2, "mgs"), (3, "mgs"), (4, "mgs"), (2, "cgs")])
def test_peer_exchange_on_one_gpu(rbg, orc, world, ortho):
    """comm = PEER (no collective library): each rank's sweep stores its maxloc record into
    every rank's record array with release-tagged stores, the wait kernel acquires the tags,
    the replicated IMGS reads the winner's column from the owner's send slot (two slots by
    tag parity).  The ranks share one stream and are driven local-on-all then finish-on-all,
    so no kernel ever waits for one that has not been launched.  Bit-identical to the oracle."""
    import torch
    S, w, tol, k_max = inputs.config1(M=3001, N=700)
    lanes = orc.CANONICAL_CGS if ortho == "cgs" else orc.CANONICAL
    o = orc.greedy(S, w, tol, k_max, lanes=lanes, ortho=ortho)
    stream = torch.cuda.Stream()
    ctxs = _peer_group(rbg, S, w, tol, k_max, world, stream.cuda_stream, ortho=ortho)
    for _ in range(k_max + 1):
        for c in ctxs:
            c.iter_local()
        for c in ctxs:
            c.iter_finish()
    res = [c.result() for c in ctxs]
    for r in res:
        assert (r.k, r.stop) == (o.k, o.stop)
        np.testing.assert_array_equal(r.pivots, o.pivots)
        np.testing.assert_array_equal(r.errors, o.errors)
        np.testing.assert_array_equal(r.nu, o.nu)
        np.testing.assert_array_equal(r.Q, o.Q)
    np.testing.assert_array_equal(np.concatenate([r.R for r in res], axis=1), o.R)
    np.testing.assert_array_equal(np.concatenate([r.r2 for r in res]), o.r2)
    if ortho == "mgs":
        # EIM works on any rank of a sharded run (the basis is replicated): the oracle's nodes
        nodes_o, B_o = orc.eim(o.Q)
        for c in ctxs:
            nodes, B = c.eim()
            np.testing.assert_array_equal(nodes, nodes_o)
            np.testing.assert_array_equal(B, B_o)
    for c in ctxs:
        c.close()


def test_peer_world1_run_and_graphs(rbg, orc):
    """A one-rank PEER context is connected at create: rbg_run and CUDA-graph batches (the
    wait kernel captured with the sweep and IMGS) give the oracle's bits; the exchange phase
    is timed as C_j."""
    S, w, tol, k_max = inputs.config1(M=2500, N=800)
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    with rbg.Context(S, w, tol, k_max, comm=rbg.COMM_PEER, rank=0, world=1) as ctx:
        ctx.set_timing(True)
        ctx.run()
        compare(ctx.result(), o)
        assert ctx.stats().t_xchg_ms > 0.0
    with rbg.Context(S, w, tol, k_max, comm=rbg.COMM_PEER, rank=0, world=1) as ctx:
        ctx.set_graph_batch(8)
        ctx.run()
        compare(ctx.result(), o)


def test_peer_setup_errors_and_timeout(rbg):
    """Unconnected PEER ranks refuse to run; local wiring needs one stream; a rank whose
    peer never publishes its record stops PEER_TIMEOUT after peer_timeout_ms instead of
    hanging (the wait kernel is bounded)."""
    import torch
    S, w, tol, k_max = inputs.config1(M=400, N=300)
    a = rbg.Context(S[:200], w, tol, 10, comm=rbg.COMM_PEER, rank=0, world=2, col_offset=0, M_global=400)
    b = rbg.Context(S[200:], w, tol, 10, comm=rbg.COMM_PEER, rank=1, world=2, col_offset=200, M_global=400)
    with pytest.raises(rbg.RbgError) as e:
        a.step(1)
    assert e.value.status == rbg.ESTATE
    with pytest.raises(rbg.RbgError) as e:
        rbg.peer_connect_local([a, b])          # two library-owned streams
    assert e.value.status == rbg.EINVAL
    assert len(a.peer_export()) == rbg.PEER_HANDLE_BYTES
    a.close()
    b.close()
    stream = torch.cuda.Stream()
    ctxs = _peer_group(rbg, S, w, tol, 10, 2, stream.cuda_stream)
    for c in ctxs:
        c.close()
    a = rbg.Context(S[:200], w, tol, 10, stream=stream.cuda_stream, comm=rbg.COMM_PEER, rank=0, world=2,
                    col_offset=0, M_global=400, peer_timeout_ms=200)
    b = rbg.Context(S[200:], w, tol, 10, stream=stream.cuda_stream, comm=rbg.COMM_PEER, rank=1, world=2,
                    col_offset=200, M_global=400, peer_timeout_ms=200)
    rbg.peer_connect_local([a, b])
    a.iter_local()                               # rank 1 never sweeps
    a.iter_finish()
    k, _, why = a.info()
    assert (k, why) == (0, "PEER_TIMEOUT")
    assert len(a.errors()) == 0                  # err_0 was never decided (no stale 0.0)
    a.close()
    b.close()


@pytest.mark.parametrize("case", ["cfg0", "cfg1", "cfg2", "cfg4", "ragged_real", "ragged_cplx"])
def test_cgs_variant_parity(rbg, orc, case):
    """Hoffmann CGSCI orthogonalisation (rbg_desc.ortho = CGS) against the oracle's CGS mode
    (lanes (32, 256)): bit for bit."""
    rng = np.random.default_rng(77)
    if case == "cfg0":
        S, w, tol, k_max = inputs.config0()
    elif case == "cfg1":
        S, w, tol, k_max = inputs.config1(M=3000, N=2000)
    elif case == "cfg2":
        S, w, tol, k_max = inputs.config2(M=2000, N=10000)
        k_max = 60
    elif case == "cfg4":
        S, w, tol, k_max, _ = inputs.config4(M=4096, N=1024, r=256)
    elif case == "ragged_real":
        S, w, tol, k_max = rng.standard_normal((300, 257)), rng.uniform(0.5, 1.5, 257), 0.0, 40
    else:
        S = rng.standard_normal((200, 4097)) + 1j * rng.standard_normal((200, 4097))
        w, tol, k_max = rng.uniform(0.5, 1.5, 4097), 0.0, 40
    g = rbg.greedy(S, w, tol, k_max, ortho="cgs")
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL_CGS, ortho="cgs")
    compare(g, o)


@pytest.mark.parametrize("case", ["cfg0", "cfg1", "cfg4", "odd_real_borrowed", "cplx_strided", "cgs"])
def test_explicit_residual_parity(rbg, orc, case):
    """Explicit residuals (Algorithm 2 in-place updates, rbg_desc.residual = EXPLICIT) against
    the oracle's explicit mode: bit for bit, and the paper's tolerances are reached."""
    import torch
    rng = np.random.default_rng(88)
    kw, okw = {}, {}
    if case == "cfg0":
        S, w, tol, k_max = inputs.config0()
    elif case == "cfg1":
        S, w, tol, k_max = inputs.config1(M=3000, N=2000)
    elif case == "cfg4":
        S, w, tol, k_max, _ = inputs.config4(M=4096, N=1024, r=256)
    elif case == "odd_real_borrowed":
        S, w, tol, k_max = rng.standard_normal((300, 257)), rng.uniform(0.5, 1.5, 257), 0.0, 60
        big = torch.full((300, 258), float("nan"), dtype=torch.float64, device="cuda")
        big[:, :257] = torch.as_tensor(S, device="cuda")
        kw["_S"] = big[:, :257]                   # padding row holds NaN: must never be read
    elif case == "cplx_strided":
        S = rng.standard_normal((200, 1000)) + 1j * rng.standard_normal((200, 1000))
        w, tol, k_max = rng.uniform(0.5, 1.5, 1000), 0.0, 50
    else:
        S, w, tol, k_max = inputs.config1(M=2000, N=800)
        kw["ortho"], okw["ortho"] = "cgs", "cgs"
    src = kw.pop("_S", S)
    lanes = orc.CANONICAL_CGS if okw.get("ortho") == "cgs" else orc.CANONICAL
    g = rbg.greedy(src, w, tol, k_max, residual="explicit", check_finite=False, **kw)
    o = orc.greedy(S, w, tol, k_max, lanes=lanes, residual="explicit", **okw)
    compare(g, o)
    if case in ("cfg0", "cfg1"):
        assert g.stop == "TOL"


@pytest.mark.parametrize("world,M,N,cplx", [(4, 5, 40, True), (3, 7, 33, False), (2, 2, 9, True)])
def test_peer_tiny_shards_until_all_selected(rbg, orc, world, M, N, cplx):
    """PEER ranks holding one or two columns each (most warps and CTAs have no column; a rank's
    record is -inf once its columns are selected) run to ALL_SELECTED with the oracle's bits."""
    import torch
    from paper_1805_06124_b200 import dist as D
    rng = np.random.default_rng(M * 31 + N)
    S = rng.standard_normal((M, N)) + (1j * rng.standard_normal((M, N)) if cplx else 0)
    w = rng.uniform(0.5, 1.5, N)
    k_max = M
    o = orc.greedy(S, w, 0.0, k_max, lanes=orc.CANONICAL)
    stream = torch.cuda.Stream()
    ctxs = []
    for p in range(world):
        off, m = D.partition(M, world, p)
        ctxs.append(rbg.Context(S[off:off + m], w, 0.0, k_max, stream=stream.cuda_stream, comm=rbg.COMM_PEER,
                                rank=p, world=world, col_offset=off, M_global=M, peer_timeout_ms=20000))
    rbg.peer_connect_local(ctxs)
    for _ in range(k_max + 2):
        for c in ctxs:
            c.iter_local()
        for c in ctxs:
            c.iter_finish()
    for c in ctxs:
        r = c.result()
        assert (r.k, r.stop) == (o.k, o.stop)
        np.testing.assert_array_equal(r.pivots, o.pivots)
        np.testing.assert_array_equal(r.errors, o.errors)
        np.testing.assert_array_equal(r.Q, o.Q)
        c.close()


@pytest.mark.parametrize("case", ["cplx", "real"])
def test_checkpoint_restore_continues_bit_for_bit(rbg, orc, tmp_path, case):
    """Checkpoint / resume (rbg_restore): a greedy stopped at k_max = 30 is saved, loaded into a
    fresh context with a larger k_max and continued; the result equals an uninterrupted run and
    the oracle bit for bit (pivots, errors, Q, R, r2, nu, rdiag, stop)."""
    if case == "cplx":
        S, w, tol, k_max = inputs.config1(M=3000, N=2000)
        k_max = 80
    else:
        S, w, tol, k_max = inputs.config0()
    full = rbg.greedy(S, w, tol, k_max)
    with rbg.Context(S, w, tol, 30) as ctx:
        ctx.run()
        assert ctx.info()[::2] == (30, "KMAX")
        rbg.save_checkpoint(ctx, str(tmp_path / "ck.npz"))
    state = rbg.load_checkpoint(str(tmp_path / "ck.npz"))
    with rbg.Context(S, w, tol, k_max) as ctx:
        import dataclasses
        with pytest.raises((rbg.RbgError, ValueError)):        # k >= k_max is refused
            ctx.restore(dataclasses.replace(state, k=k_max))
        ctx.restore(state)
        ctx.run()
        g = ctx.result()
        with pytest.raises(rbg.RbgError) as e:
            ctx.restore(state)                                # not a fresh context any more
        assert e.value.status == rbg.ESTATE
    o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
    for ref in (full, o):
        assert (g.k, g.stop) == (ref.k, ref.stop)
        for key in ("pivots", "errors", "Q", "R", "r2", "nu", "rdiag"):
            np.testing.assert_array_equal(getattr(g, key), getattr(ref, key))
