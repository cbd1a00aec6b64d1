"""Out-of-bounds write detection on the GPU (compute-sanitizer is closed on this pool).

With canaries on, every device buffer the library allocates carries a 256-byte 0xA5 tail
that is checked when the buffer is freed and on demand.  Every kernel family runs on small
cases -- both sweeps (init / coefficient, complex / real odd N), the MGS and CGS IMGS, the
explicit-residual sweep, validation, enrichment, Gram, Jacobi + reconstruction, EIM, the
EXTERNAL and PEER exchanges -- and no canary may be touched.  A deliberate one-byte overrun
of a library buffer must be reported.
"""
import numpy as np
import pytest

from paper_1805_06124_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture()
def rbg():
    import torch
    assert torch.cuda.is_available()
    from paper_1805_06124_b200 import rbg as R
    R.set_canary(True)
    yield R
    R.set_canary(False)


def _families(rbg):
    import torch
    S, w, tol, _ = inputs.config1(M=700, N=300)
    for kw in ({}, {"ortho": "cgs"}, {"residual": "explicit"}):
        with rbg.Context(S, w, tol, 40, **kw) as ctx:
            ctx.run()
            ctx.result()
            if not kw:
                ctx.validate(S[:50], coeffs=True)
                ctx.gram()
                ctx.reconstruct(1e-3)
                ctx.eim()
                ctx.add_columns(S[:20] * 1.5)
                ctx.run()
    Sr = np.random.default_rng(1).standard_normal((100, 257))     # real, odd N (padding row)
    rbg.greedy(Sr, None, 0.0, 30)
    rbg.greedy(Sr, None, 0.0, 30, residual="explicit")
    ext = [rbg.Context(S[p * 350:(p + 1) * 350], w, tol, 20, comm=rbg.COMM_EXTERNAL, rank=p, world=2,
                       col_offset=p * 350, M_global=700) for p in range(2)]
    for _ in range(21):
        for c in ext:
            c.iter_local()
        rbg.emulate_allgather(ext)
        for c in ext:
            c.iter_finish()
    for c in ext:
        c.close()
    st = torch.cuda.Stream()
    peer = [rbg.Context(S[p * 350:(p + 1) * 350], w, tol, 20, stream=st.cuda_stream, comm=rbg.COMM_PEER,
                        rank=p, world=2, col_offset=p * 350, M_global=700) for p in range(2)]
    rbg.peer_connect_local(peer)
    for _ in range(21):
        for c in peer:
            c.iter_local()
        for c in peer:
            c.iter_finish()
    for c in peer:
        c.close()


def test_no_kernel_writes_out_of_bounds(rbg):
    before, _ = rbg.canary_violations()
    _families(rbg)
    n, msg = rbg.canary_violations()
    assert n == before, msg


def test_overrun_is_detected(rbg):
    from cuda.bindings import runtime as cudart
    S, w, tol, _ = inputs.config1(M=64, N=100)
    before, _ = rbg.canary_violations()
    ctx = rbg.Context(S, w, tol, 4, comm=rbg.COMM_EXTERNAL, rank=0, world=1)
    send, _, nbytes = ctx.xchg_buffers()
    err, = cudart.cudaMemset(send + nbytes, 0, 1)     # one byte past the send slot
    assert err == cudart.cudaError_t.cudaSuccess
    ctx.close()                                        # checked at free
    n, msg = rbg.canary_violations()
    assert n == before + 1 and "past the end" in msg
