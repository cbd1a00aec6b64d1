#!/usr/bin/env python
"""IMGS / small-config timings for round 2, one JSON line per measurement.

    python scripts/imgs_probe_r2.py [tag]

  * whole greedy of configs 0, 1, 4 (MGS, recurrence) through rbg_run -- the device loop
    (conditional WHILE graph) with programmatic dependent launches unless RBG_NO_PDL is set --
    timed with CUDA events around rbg_run on the library's stream; us per iteration and the
    no-op iterations launched past the stop (rbg_stats.noop_iters);
  * per-phase events (timing mode, plain launches) on the same configs: mean IMGS and sweep
    per iteration;
  * IMGS time vs k on config 2's recipe at 40,960 columns (k_max 300), per MGS step.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

TAG = sys.argv[1] if len(sys.argv) > 1 else ("nopdl" if os.environ.get("RBG_NO_PDL") else "pdl")


def emit(d):
    d["tag"] = TAG
    print(json.dumps(d), flush=True)


def whole(cfg, S, w, tol, k_max):
    St = torch.as_tensor(S, device="cuda")
    stream = torch.cuda.Stream()
    best = None
    for rep in range(3):
        with rbg.Context(St, w, tol, k_max, stream=stream.cuda_stream) as ctx:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.run()
            e1.record(stream)
            e1.synchronize()
            k, _, why = ctx.info()
            ms = e0.elapsed_time(e1)
            noop = ctx.stats().noop_iters
        if rep > 0 and (best is None or ms < best[2]):
            best = (k, why, ms, noop)
    k, why, ms, noop = best
    emit({"what": "whole_greedy_rbg_run", "config": cfg, "k": k, "stop": why, "ms": ms,
          "us_per_iter": ms * 1e3 / (k + 1), "noop_iters": noop})
    with rbg.Context(St, w, tol, k_max, stream=stream.cuda_stream) as ctx:
        ctx.set_timing(True)
        ctx.run()
        k = ctx.info()[0]
        sw, xc, im = ctx.timings(k + 1)
        st = ctx.stats()
    emit({"what": "phases_timing_mode", "config": cfg, "k": k, "imgs_us_mean": float(np.nanmean(im)) * 1e3,
          "sweep_us_mean": float(np.nanmean(sw[:k])) * 1e3, "gap_ms_total": st.t_gap_ms,
          "total_ms": st.t_total_ms, "us_per_iter_events": st.t_total_ms * 1e3 / (k + 1)})


def scaling():
    M, K, N = 40960, 300, 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(M, 2, spin=True)
    S = torch.empty((M, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
    with rbg.Context(S, w, 0.0, K) as ctx:
        ctx.set_timing(True)
        ctx.run()
        k = ctx.info()[0]
        sw, xc, im = ctx.timings(k)
        nu = ctx.nu()
    for i in [1, 2, 5, 10, 25, 50, 100, 150, 200, 250, k - 1]:
        if i < k:
            emit({"what": "imgs_vs_k", "k": i, "nu": int(nu[i]), "imgs_us": im[i] * 1e3,
                  "us_per_mgs_step": im[i] * 1e3 / max(nu[i] * i, 1)})


def main():
    for cfg, args in ((0, inputs.config0()), (1, inputs.config1()), (4, inputs.make(4))):
        whole(cfg, *args)
    scaling()


if __name__ == "__main__":
    main()
