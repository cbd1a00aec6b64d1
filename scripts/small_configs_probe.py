#!/usr/bin/env python
"""Whole-greedy device time of the small configs (0, 1, 4), warm (the greedy is run once
before the timed run, so module loading is excluded), with the per-phase split from the
library's CUDA events (rbg_set_timing).  Prints one JSON line per config; run it under
different RBG_IMGS_CTAS values to compare IMGS cluster sizes."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402


def run(S, w, tol, k_max):
    St = torch.as_tensor(S, device="cuda")
    stream = torch.cuda.Stream()
    out = None
    for rep in range(2):
        with rbg.Context(St, w, tol, k_max, stream=stream.cuda_stream) as ctx:
            ctx.set_timing(True)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.step(k_max + 1)
            e1.record(stream)
            e1.synchronize()
            k, _, why = ctx.info()
            sw, xc, im = ctx.timings(k)
            out = {"k": k, "stop": why, "ms_total": e0.elapsed_time(e1), "us_per_iter": e0.elapsed_time(e1) / k * 1e3,
                   "sweep_us_avg": float(np.mean(sw)) * 1e3, "imgs_us_avg": float(np.mean(im)) * 1e3}
    return out


def main():
    cases = {0: inputs.config0(), 1: inputs.config1(), 4: inputs.make(4)}
    for cfg, (S, w, tol, k_max) in cases.items():
        r = run(S, w, tol, k_max)
        print(json.dumps({"config": cfg, "imgs_ctas": os.environ.get("RBG_IMGS_CTAS", "16"), **r}), flush=True)


if __name__ == "__main__":
    main()
