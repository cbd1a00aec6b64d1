#!/usr/bin/env python
"""A/B of a library environment switch on the whole greedy of configs 0, 1, 4.

    python scripts/env_ab_probe.py VAR v1 v2 ...   # one subprocess per value, alternated twice

Each value runs scripts/imgs_probe_r2.py's whole-greedy measurement (rbg_run, device loop,
best of two timed runs) in a fresh process (the library reads its switches once); the tag is
VAR=value.  Used for RBG_L2_KEEP_MB (an L2-resident column prefix, removed after its A/B:
profiles/r02/l2keep_ab.txt) and RBG_LASTWAVE_PF (a last-wave L2 prefetch, likewise removed:
profiles/r02/lastwave_ab.txt).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

CHILD = r"""
import sys
sys.path.insert(0, %r)
import imgs_probe_r2 as P
from paper_1805_06124_b200 import inputs
for cfg, args in ((0, inputs.config0()), (1, inputs.config1()), (4, inputs.make(4))):
    P.whole(cfg, *args)
"""

if __name__ == "__main__":
    var, values = sys.argv[1], sys.argv[2:]
    for rep in (1, 2):
        for v in values:
            env = dict(os.environ, **{var: v})
            subprocess.run([sys.executable, "-c", CHILD % HERE, f"{var}={v}"], env=env, check=True,
                           cwd=os.path.dirname(HERE))
