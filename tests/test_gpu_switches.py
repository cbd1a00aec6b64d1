"""Every A/B switch of round 2 gives the default path's bits: the IMGS basis
pipe by bulk copies instead of 4D tensor-map TMA (RBG_IMGS_BULK), no programmatic dependent
launch (RBG_NO_PDL), rbg_run polling instead of the conditional-graph device loop
(RBG_NO_DEVICE_LOOP), no tail prefetch in the sweep (RBG_NO_TAIL_PF), the 16-CTA IMGS cluster
instead of the 1-4-CTA one at nvec <= 512 (RBG_IMGS_SMALL=0).  The switches are read
once per process, so each variant runs in a subprocess on the same inputs; the default run is
also checked against the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SWITCHES = ["RBG_IMGS_BULK", "RBG_NO_PDL", "RBG_NO_DEVICE_LOOP", "RBG_NO_TAIL_PF", "RBG_IMGS_SMALL"]

_CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_1805_06124_b200 import rbg
S = np.load({s!r}); w = np.load({w!r})
r = rbg.greedy(S, w, {tol!r}, {k_max})
np.savez({out!r}, k=r.k, pivots=r.pivots, errors=r.errors, Q=r.Q, R=r.R, nu=r.nu, r2=r.r2)
"""


def test_switches_give_the_default_bits(orc, tmp_path):
    from paper_1805_06124_b200 import inputs, rbg
    cases = {"n10000": inputs.config2(M=3000, N=10000)[:2] + (0.0, 40),   # MAXV = 5: the TMA basis pipe
             "cfg1": inputs.config1(M=3000, N=2000),
             "cfg0": inputs.config0()}                                        # nvec = 128: one-CTA IMGS
    for name, (S, w, tol, k_max) in cases.items():
        s_path, w_path = tmp_path / f"{name}_S.npy", tmp_path / f"{name}_w.npy"
        np.save(s_path, S)
        np.save(w_path, w)
        g = rbg.greedy(S, w, tol, k_max)
        o = orc.greedy(S, w, tol, k_max, lanes=orc.CANONICAL)
        assert (g.k, g.stop) == (o.k, o.stop)
        for key in ("pivots", "errors", "Q", "R", "nu", "r2"):
            np.testing.assert_array_equal(getattr(g, key), getattr(o, key))
        for sw in SWITCHES:
            out = tmp_path / f"{name}_{sw}.npz"
            code = _CODE.format(root=ROOT, s=str(s_path), w=str(w_path), tol=tol, k_max=k_max, out=str(out))
            val = "0" if sw == "RBG_IMGS_SMALL" else "1"   # RBG_IMGS_SMALL=0: the 16-CTA cluster at small N
            p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **{sw: val}), capture_output=True,
                               text=True, timeout=600)
            assert p.returncode == 0, (sw, p.stderr[-2000:])
            c = np.load(out)
            assert int(c["k"]) == g.k, sw
            for key in ("pivots", "errors", "Q", "R", "nu", "r2"):
                np.testing.assert_array_equal(c[key], getattr(g, key), err_msg=f"{name} {sw} {key}")
