#!/usr/bin/env python
"""Measurements of the NEXT rows (DESIGN.md f-1, f-3) on the config-2 basis (1 x B200).

    python scripts/bench_next.py [--cols 409600] [--val-cols 40960] [--k 300]

After the k-iteration greedy on the device-generated config-2 matrix:
  * validation of an independent chirp block: the blocked coefficient kernel (one pass, FP64
    FLOP/s against the derived FP64 peak) and, for comparison, the k + 1 streaming sweep
    passes it replaced (RBG_COEFF=passes; HBM GB/s against MEASURED_PEAKS.json);
  * enrichment step: rbg_add_columns of 4,096 columns (copy + k coefficient passes);
  * Algorithm 4 reconstruction: Gram (FP64 FLOP/s against the derived FP64 peak), Jacobi,
    X = Q V; total;
  * greedy EIM nodes of the k-vector basis.
Beside each GPU number, the CPU oracle (oracle/, as it stands, all host cores) on the same
data (a column sample for validation, scaled), so every NEXT row is measured against its
roofline with the oracle timed beside it.
Prints one JSON line.  Timed with CUDA events / wall clock around blocking ABI calls.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (the CPU baseline legs only)
from paper_1805_06124_b200 import inputs, rbg  # noqa: E402

FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cols", type=int, default=409600)
    p.add_argument("--val-cols", type=int, default=40960)
    p.add_argument("--k", type=int, default=300)
    a = p.parse_args()
    N = 10000
    t = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(a.cols, 2, spin=True)
    S = torch.empty((a.cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(S, t, w, q, chi, psi, spin=True)
    qv, cv, pv = inputs.chirp_params(a.val_cols, 12, spin=True)
    V = torch.empty((a.val_cols, N), dtype=torch.complex128, device="cuda")
    rbg.gen_chirp(V, t, w, qv, cv, pv, spin=True)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    out = {"workload": f"config2 basis k={a.k} on {a.cols} x {N}; validation block {a.val_cols} x {N}"}
    with rbg.Context(S, w, 0.0, a.k) as ctx:
        ctx.run()
        torch.cuda.synchronize()
        # ---- f-1 validation (warm once)
        ctx.validate(V[:1024])
        t0 = time.perf_counter()
        err = ctx.validate(V)
        tv = time.perf_counter() - t0
        os.environ["RBG_COEFF"] = "passes"          # the k streaming coefficient sweeps
        ctx.validate(V[:1024])
        t0 = time.perf_counter()
        err_p = ctx.validate(V)
        tvp = time.perf_counter() - t0
        del os.environ["RBG_COEFF"]
        assert np.array_equal(err, err_p)
        bytes_v = (a.k + 1) * (a.val_cols * N * 16 + a.val_cols * 32)
        flops_v = 8.0 * a.k * a.val_cols * N                       # the coefficient block
        out["validate"] = {"s": tv, "kernel": "k_coeff_block (one blocked pass, coeff.cu) + 1 norm sweep",
                           "TFLOPs": flops_v / tv / 1e12,
                           "frac_of_fp64_peak": flops_v / tv / 1e12 / FP64_PEAK_TFLOPS,
                           "passes_s": tvp, "passes": a.k + 1, "passes_GBps": bytes_v / tvp / 1e9,
                           "passes_frac_of_measured_hbm": bytes_v / tvp / 1e9 / peaks["hbm_gbs"],
                           "speedup_vs_passes": tvp / tv, "bit_identical_to_passes": True,
                           "max_err": float(err.max()), "median_err": float(np.median(err)),
                           "note": "wall time of the blocking call: includes the device copy and NaN scan of V"}
        # ---- f-3 reconstruction
        ctx.reconstruct(0.0)               # warm (module load, cooperative launch setup)
        t0 = time.perf_counter()
        G = ctx.gram()
        tg = time.perf_counter() - t0
        t0 = time.perf_counter()
        sigma, kr, X = ctx.reconstruct(1e-3)
        tr = time.perf_counter() - t0
        pairs = a.k * (a.k + 1) / 2
        flops = pairs * a.cols * 8
        out["reconstruct"] = {"gram_s": tg, "gram_TFLOPs": flops / tg / 1e12,
                              "gram_frac_of_fp64_peak": flops / tg / 1e12 / FP64_PEAK_TFLOPS,
                              "fp64_peak_TFLOPs_derived": FP64_PEAK_TFLOPS,
                              "total_s": tr, "kr": kr, "sigma_1": float(sigma[0]),
                              "sigma_k": float(sigma[-1])}
        # ---- f-2 EIM nodes
        ctx.eim()
        t0 = time.perf_counter()
        nodes, B = ctx.eim()
        out["eim"] = {"s": time.perf_counter() - t0, "k": int(len(nodes)),
                      "cond_B": float(np.linalg.cond(B))}
        # ---- CPU oracle beside each row (same data; validation on a column sample, scaled)
        Qh = ctx.basis()
        Rh = ctx.R()
        res = ctx.result(full=False)
        res.Q, res.R = Qh, Rh
        # ---- f-1 enrichment step, timed before the oracle legs (their OpenMP worker threads
        # spin after each parallel region and delayed the appends' host-side calls 10-50x)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.add_columns(V[:4096])
        out["add_columns_4096_s"] = time.perf_counter() - t0     # first append: R grows (+1/8 slack)
        t0 = time.perf_counter()
        ctx.add_columns(V[4096:8192])
        out["add_columns_4096_again_s"] = time.perf_counter() - t0   # within R's slack: in place
        ncores = len(os.sched_getaffinity(0))
        ns = 2048
        Vh = V[:ns].cpu().numpy()
        t0 = time.perf_counter()
        O.validate(Qh, Vh, w)
        tvo = (time.perf_counter() - t0) * a.val_cols / ns
        out["validate"]["oracle_s"] = tvo
        out["validate"]["oracle_sample"] = f"{ns} of {a.val_cols} columns, scaled"
        t0 = time.perf_counter()
        O.gram(Rh)
        tgo = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.reconstruct(res, 1e-3)
        tro = time.perf_counter() - t0
        out["reconstruct"].update({"oracle_gram_s": tgo, "oracle_total_s": tro,
                                   "jacobi_and_x_s": tr - tg,
                                   "note": "oracle eigen-step = LAPACK eigh (a library step of the oracle)"})
        t0 = time.perf_counter()
        O.eim(Qh)
        out["eim"].update({"oracle_s": time.perf_counter() - t0,
                           "us_per_step": out["eim"]["s"] / max(len(nodes), 1) * 1e6,
                           "bound": "latency (k dependent argmax-over-N steps, one forward substitution each)"})
        out["oracle_cores"] = ncores

    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
