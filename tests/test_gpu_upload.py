"""rbg_create's chunked upload: with the chunk forced down to a few columns, the
finiteness scan of every chunk reports the first non-finite entry in column-major order with
its global (row, col), host and device-copy sources, and a finite input still gives the
oracle's bits.  The chunk size is read once per process, so each case runs in a subprocess."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CODE = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1805_06124_b200 import rbg
S = np.load({s!r})
src = torch.as_tensor(S, device="cuda") if {dev!r} else S
try:
    r = rbg.greedy(src, None, 0.0, 8, borrow=False)
    np.savez({out!r}, ok=1, pivots=r.pivots, errors=r.errors, Q=r.Q)
except rbg.RbgError as e:
    np.savez({out!r}, ok=0, msg=str(e), status=e.status)
"""


def _run(tmp_path, S, dev, name):
    s_path, out = tmp_path / f"{name}.npy", tmp_path / f"{name}.npz"
    np.save(s_path, S)
    code = _CODE.format(root=ROOT, s=str(s_path), dev=dev, out=str(out))
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RBG_UPLOAD_CHUNK_COLS="3"),
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("dev", [False, True])
@pytest.mark.parametrize("cplx", [False, True])
def test_chunked_upload_scan_and_bits(orc, tmp_path, dev, cplx):
    rng = np.random.default_rng(7 + cplx)
    M, N = 20, 33
    S = rng.standard_normal((M, N)) + (1j * rng.standard_normal((M, N)) if cplx else 0)
    r = _run(tmp_path, S, dev, "finite")
    assert int(r["ok"]) == 1
    o = orc.greedy(S, np.ones(N), 0.0, 8, lanes=orc.CANONICAL)
    np.testing.assert_array_equal(r["pivots"], o.pivots)
    np.testing.assert_array_equal(r["errors"], o.errors)
    np.testing.assert_array_equal(r["Q"], o.Q)
    bad = S.copy()
    bad[17, 5] = np.nan          # column 17: chunk 5 of the 3-column chunks
    bad[13, 30] = np.inf         # column 13 (chunk 4), row 30: the first in column-major order
    r = _run(tmp_path, bad, dev, "nonfinite")
    assert int(r["ok"]) == 0
    assert "row 30, col 13" in str(r["msg"]), str(r["msg"])   # column 13 comes before column 17
