#!/usr/bin/env python
"""Whole-greedy timings for the small BASELINE.json configs (0, 1, 4) on one B200.

    python scripts/bench_configs.py

For each config: host-generated input (inputs.py), uploaded once; the full greedy to its
stop reason timed on the device (CUDA events around rbg_step on the library's stream),
with plain launches and with CUDA-graph batches of 16 iterations, for both orthogonalisation
variants.  One JSON line per (config, variant).
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402


def run(S, w, tol, k_max, graph, ortho, residual="recurrence"):
    St = torch.as_tensor(S, device="cuda")
    stream = torch.cuda.Stream()
    with rbg.Context(St, w, tol, k_max, stream=stream.cuda_stream, ortho=ortho, residual=residual) as ctx:
        if graph:
            ctx.set_graph_batch(16)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.step(k_max + 1)
        e1.record(stream)
        e1.synchronize()
        k, _, why = ctx.info()
        return k, why, e0.elapsed_time(e1)


def main():
    cases = {0: inputs.config0(), 1: inputs.config1(), 4: inputs.make(4)}
    for cfg, (S, w, tol, k_max) in cases.items():
        for residual in ("recurrence", "explicit"):
            for ortho in ("mgs", "cgs"):
                for graph in (False, True):
                    run(S, w, tol, k_max, graph, ortho, residual)          # warm (module load, graph build)
                    k, why, ms = run(S, w, tol, k_max, graph, ortho, residual)
                    print(json.dumps({"config": cfg, "shape": list(S.shape[::-1]), "dtype": str(S.dtype),
                                      "residual": residual, "ortho": ortho, "cuda_graph": graph, "k": k,
                                      "stop": why, "ms_total": ms, "iters_per_s": k / (ms / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
