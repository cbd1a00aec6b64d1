#!/usr/bin/env python
"""Plain-mode agreement depth (SURVEY §8(c) parity contract item 2; BASELINE.md CPU plan):
the CPU oracle with textbook sequential sums (lanes (1, 1), "plain mode") against the
canonical lane counts (the GPU's arithmetic) on configs 0, 1 and 4.  Reports the first
iteration d where the pivots differ, the greedy error there relative to err_0, both runs'
k and stop reasons, and the largest |err_k| difference before d.  Oracle only (CPU)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1805_06124_b200 import inputs  # noqa: E402


def main():
    for name, (S, w, tol, k_max) in [("config0", inputs.config0()), ("config1", inputs.config1()),
                                     ("config4", inputs.make(4))]:
        c = O.greedy(S, w, tol, k_max, lanes=O.CANONICAL)
        p = O.greedy(S, w, tol, k_max, lanes=(1, 1))
        n = min(c.k, p.k)
        diff = np.nonzero(np.asarray(c.pivots[:n]) != np.asarray(p.pivots[:n]))[0]
        d = int(diff[0]) if len(diff) else n
        e0 = float(c.errors[0])
        de = float(np.max(np.abs(np.asarray(c.errors[:d + 1]) - np.asarray(p.errors[:d + 1])))) if d > 0 else 0.0
        # SURVEY's acceptance test for a mismatch at d: the plain oracle's residuals of the two
        # candidates differ by <= 1e3 * eps * max ||s||^2
        gap = None
        if d < n:
            ps = O.greedy(S, w, tol, k_max, lanes=(1, 1), max_iters=d)
            jc, jp = int(c.pivots[d]), int(p.pivots[d])
            gap = abs(float(ps.r2[jc]) - float(ps.r2[jp])) / (e0 * e0)
        print(json.dumps({"config": name, "canonical": {"k": int(c.k), "stop": c.stop},
                          "plain": {"k": int(p.k), "stop": p.stop}, "agreement_depth": d,
                          "err_at_d_rel": float(c.errors[d]) / e0 if d < len(c.errors) else None,
                          "max_abs_err_diff_before_d": de, "err0": e0,
                          "candidate_gap_rel_at_d": gap,
                          "acceptable": gap is None or gap <= 1e3 * 2.0 ** -52}), flush=True)


if __name__ == "__main__":
    main()
