#!/usr/bin/env python
"""A/B of the sweep's L2-resident column prefix (RBG_L2_KEEP_MB) on configs 0, 1, 4.

    python scripts/l2keep_probe.py 0 32 64 96     # one subprocess per budget, alternated twice

(The experimental RBG_L2_KEEP_MB knob was removed after this A/B: no gain.)
Each budget runs scripts/imgs_probe_r2.py's whole-greedy measurement (rbg_run, device loop,
best of two timed runs) in a fresh process (the library reads the variable once); the tag is
the budget in MB.  Same bits either way: only the L2 eviction priority of the loads changes.
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
    budgets = sys.argv[1:] or ["0", "64"]
    for rep in (1, 2):
        for mb in budgets:
            env = dict(os.environ, RBG_L2_KEEP_MB=mb)
            code = CHILD % HERE
            subprocess.run([sys.executable, "-c", code, f"keep{mb}"], env=env, check=True,
                           cwd=os.path.dirname(HERE))
