#!/usr/bin/env python
"""bench.py -- the RB-greedy hot path (arXiv 1805.06124) on B200, one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1, one rank per GPU)

Workload (BASELINE.json config 2; config 3 weak scaling for N > 1): complex fp64 chirp
snapshots, N = 10,000 rows x 409,600 columns PER GPU (65.5 GB per GPU, generated on the
device), Simpson weights, tol 0, k_max 300.  One step = one greedy iteration (pivot
decision + IMGS + fused sweep over all columns).  W warm-up iterations (plus sweep 0) run
untimed, then exactly K iterations are timed with CUDA events on the library's stream,
max over ranks.  Inputs (65.5 GB) exceed the 126 MB L2, so no flush is needed.

``value`` is whole-job throughput: greedy iterations/s times the number of 409,600-column
shards (= plain iterations/s at N = 1, the metric BASELINE.json quotes).  The JSON line
also carries the fused sweep's roofline (HBM bytes per launch / event-timed duration,
against MEASURED_PEAKS.json), the CPU oracle baseline on a bounded sample, an end-to-end
number through the C ABI with host buffers, and the SM clocks seen during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "greedy iterations/s and achieved HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs"
N_ROWS = 10_000
M_PER_GPU = 409_600
K_MAX = 300
CPU_SAMPLE_COLS = 16_384
SPEC_HBM_GBS = 8000.0          # B200 datasheet HBM3e bandwidth (context)
# measured read-only ceiling of the sweep's own access pattern on this pool's B200s (one warp
# per 160 KB column, 16-byte loads, columns dealt dynamically from a grid-wide counter, best
# of the T/U/occupancy variants): scripts/hbm_probe2.cu, profiles/r01/hbm_probe2.txt
READ_STREAM_GBS = 7465.3


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=K_MAX - 3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rows", type=int, default=N_ROWS)
    p.add_argument("--cols-per-gpu", type=int, default=M_PER_GPU)
    p.add_argument("--strong-cols", type=int, default=0,
                   help="strong scaling: this many columns in total, split over the GPUs "
                        "(BASELINE config 3: 1,638,400 at 2/4/8 GPUs); default weak scaling")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--graph-batch", type=int, default=0)
    p.add_argument("--ortho", default="mgs", choices=["mgs", "cgs"],
                   help="IMGS variant: the paper's MGSCI (default) or Hoffmann CGSCI")
    p.add_argument("--residual", default="recurrence", choices=["recurrence", "explicit"],
                   help="column residuals: the paper's recurrence (default) or Algorithm 2 updates")
    p.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                   help="N > 1 exchange: records/pivot column over NVLink inside the kernels (default) "
                        "or one ncclAllGather per iteration")
    return p.parse_args()


# ----------------------------------------------------------------------------- helpers

class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "-i", str(device),
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(", ") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows)}


def peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


def ncu_traffic():
    """dram bytes per sweep launch from the committed ncu --set full capture, if any."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "sweep_traffic.json")))["traffic_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def cpu_sample(cols: int, iters: int, cfg: int = 2, S=None):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: the first `cols`
    columns of the device matrix when given (the same bytes the GPU streamed), else the same
    recipe generated on the host."""
    from oracle import oracle as O
    from paper_1805_06124_b200 import inputs
    if S is None:
        S, w, _, _ = inputs.config2(M=cols, N=N_ROWS, cfg=cfg)
    else:
        w = inputs.simpson_weights(N_ROWS)
    t0 = time.perf_counter()
    r = O.greedy(S, w, 0.0, max(K_MAX, iters), lanes=O.CANONICAL, max_iters=iters)
    wall = time.perf_counter() - t0
    return r, wall


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def full_iter_seconds(r, lo: int, hi: int, cols: int, m_full: int) -> float:
    """Per-iteration oracle time on the full workload from a column sample: the column sweep
    and pivot search scale with the column count, IMGS does not."""
    t_it = np.asarray(r.t_iter[lo:hi])
    t_im = np.asarray(r.t_imgs[lo:hi])
    return float(np.mean((t_it - t_im) * (m_full / cols) + t_im))


# ----------------------------------------------------------------------------- reference arm

def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = a.gpus
    m_full = a.cols_per_gpu * world
    W, K = a.warmup, a.steps
    r, wall = cpu_sample(CPU_SAMPLE_COLS, W + K)
    t = full_iter_seconds(r, W, W + K, CPU_SAMPLE_COLS, m_full)
    val = 1.0 / t * (m_full / M_PER_GPU)     # the same whole-job unit as our arm
    cores = oracle_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "it/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if a.strong_cols else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(a, world),
        "cpu_baseline": {"value": val, "unit": "it/s", "cores": cores, "kind": "oracle",
                         "sample": f"CPU oracle (canonical lanes) on {CPU_SAMPLE_COLS} of "
                                   f"{m_full} columns x {a.rows} rows, iterations {W}..{W + K - 1}; "
                                   "sweep+pivot time scaled by the column ratio, IMGS as measured"},
        "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(a, world):
    if getattr(a, "strong_cols", 0):
        wl = f"config3 strong: 10,000 x {a.strong_cols} over {world} GPUs ({a.cols_per_gpu} per GPU), k_max 300"
    elif world == 1:
        wl = "config2: complex fp64 chirp snapshots 10,000 x 409,600 (65.5 GB), k_max 300"
    else:
        wl = f"config3 weak: 10,000 x 409,600 per GPU x {world} GPUs, k_max 300"
    return {"workload": wl,
            "rows": a.rows, "cols_per_gpu": a.cols_per_gpu, "cols_global": a.cols_per_gpu * world,
            "k_window": [a.warmup, a.warmup + a.steps], "parallelism": f"column-sharded x{world}",
            "l2": "inputs (65.5 GB/GPU) >> 126 MB L2; no flush",
            "ortho": getattr(a, "ortho", "mgs"), "residual": getattr(a, "residual", "recurrence"),
            "exchange": (getattr(a, "comm", "peer") if world > 1 else "none"),  # as requested
            "value_unit": "greedy iterations/s x (cols_global / 409,600) -- plain it/s at 1 GPU"}


# ----------------------------------------------------------------------------- our arm

def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_1805_06124_b200 import dist as D
    from paper_1805_06124_b200 import inputs
    from paper_1805_06124_b200 import rbg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    W, K = a.warmup, a.steps
    if W < 3:
        raise SystemExit("--warmup must be >= 3")
    k_max = max(K_MAX, W + K)
    N, M_loc = a.rows, a.cols_per_gpu
    M_glob = M_loc * world
    cfg = 2 if world == 1 else 3

    # ---- synthetic input, generated on the device
    t_grid = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(M_glob, cfg, spin=True)
    off, m_loc = D.partition(M_glob, world, rank)
    assert m_loc == M_loc
    sl = slice(off, off + M_loc)
    S = torch.empty((M_loc, N), dtype=torch.complex128, device=dev)
    rbg.gen_chirp(S, t_grid, w, q[sl], chi[sl], psi[sl], spin=True)

    stream = torch.cuda.Stream(dev)                 # the library enqueues on this stream
    torch.cuda.set_stream(stream)

    def make_ctx(comm):
        nccl_id = D.nccl_unique_id() if comm == rbg.COMM_NCCL else None
        ctx = rbg.Context(S, w, 0.0, k_max, stream=stream.cuda_stream, comm=comm, rank=rank,
                          world=world, col_offset=off, M_global=M_glob, nccl_id=nccl_id, ortho=a.ortho,
                          residual=a.residual, peer_timeout_ms=20000)
        if comm == rbg.COMM_PEER:
            D.connect_peers(ctx)
        ctx.set_timing(True)
        if a.graph_batch:
            ctx.set_graph_batch(a.graph_batch)
        ctx.step(W)                                  # warm-up: sweep 0 + W iterations
        torch.cuda.synchronize()
        return ctx

    comm = rbg.COMM_NONE
    if world > 1:
        comm = rbg.COMM_PEER if a.comm == "peer" else rbg.COMM_NCCL
    fallback = None
    if comm == rbg.COMM_PEER:
        # the PEER exchange needs CUDA IPC between the ranks' processes: if any rank cannot map
        # its peers or the warm-up timed out, every rank falls back to the NCCL exchange
        ok, ctx = True, None
        try:
            ctx = make_ctx(comm)
            ok = ctx.info()[2] != "PEER_TIMEOUT"
        except rbg.RbgError as e:
            ok, fallback = False, str(e)
        t = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if not bool(t.item()):
            if ctx is not None:
                ctx.close()
            fallback = fallback or "PEER warm-up failed on some rank"
            comm = rbg.COMM_NCCL
            ctx = make_ctx(comm)
    else:
        ctx = make_ctx(comm)

    # ---- exactly K timed iterations
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.step(K)
    e1.record(stream)
    e1.synchronize()
    clocks = clk.stop()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = D.max_over_ranks(e0.elapsed_time(e1), device=dev)
    k, _, why = ctx.info()
    if k != W + K:
        raise SystemExit(f"greedy stopped early ({why} at k={k}); the timed steps were not all real")
    sweep_ms, xchg_ms, imgs_ms = ctx.timings(W + K)
    # iteration t's sweep uses q_{t-1}: timed iterations W..W+K-1 -> sweeps W-1..W+K-2
    sw = sweep_ms[W - 1:W + K - 1]
    im = imgs_ms[W:W + K]
    xc = xchg_ms[W:W + K]
    errs = ctx.errors()
    replicas = None
    if world > 1:
        # the replicated IMGS must leave bit-identical pivots / errors / basis on every rank
        # (SURVEY §5 integrity check): compare a hash of their bits across the ranks
        import hashlib
        hsh = hashlib.sha256()
        for arr in (ctx.pivots(), errs, ctx.basis()):
            hsh.update(np.ascontiguousarray(arr).tobytes())
        replicas = len(set(D.all_gather_bytes(hsh.hexdigest()))) == 1
    ctx.close()

    it_s = K / (ms / 1e3)
    value = it_s * (M_glob / M_PER_GPU)
    bytes_sweep = N * M_loc * 16 + M_loc * (8 + 8 + 16)      # DESIGN.md "Roofline" per launch
    if a.residual == "explicit":
        bytes_sweep += 2 * N * M_loc * 16                     # + re-read and write-back of V
    sweep_avg_s = float(np.mean(sw)) / 1e3
    achieved = bytes_sweep / sweep_avg_s / 1e9
    pk = peaks()
    peak = pk.get("hbm_gbs") or 6650.0
    roof = {"kernel": "k_sweep_dyn (fused coefficient sweep + r2 update + maxloc, dynamically scheduled columns)", "bound": "hbm",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if pk.get("hbm_gbs") else "fallback 6.65 TB/s",
            "traffic": ncu_traffic(), "algorithmic_bytes_per_launch": bytes_sweep,
            "sweep_ms_avg": sweep_avg_s * 1e3,
            # SURVEY 8(d) quotes the median sweep over iterations k >= 3
            "sweep_ms_median": float(np.median(sw)),
            "achieved_at_median_gbs": bytes_sweep / (float(np.median(sw)) / 1e3) / 1e9,
            "share_of_step": float(np.sum(sw) / ms),
            # the same achieved bandwidth against the datasheet figure and the
            # measured read-only ceiling of the same access pattern
            "frac_of_spec_8tbs": achieved / SPEC_HBM_GBS,
            "read_stream_ceiling_gbs": READ_STREAM_GBS,
            "frac_of_read_stream_ceiling": achieved / READ_STREAM_GBS}

    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "strong" if a.strong_cols else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (device-generated chirps, BASELINE.json config 2/3 recipe)",
        "config": config_dict(a, world), "iters_per_s": it_s,
        "hbm_gbs_per_gpu": achieved, "hbm_gbs_total": achieved * world,
        "phase_ms_avg": {"sweep": float(np.mean(sw)), "xchg": float(np.mean(xc)), "imgs": float(np.mean(im))},
        # the paper's identity T_j = T_pivot + C_j + T_IMGS, summed over the
        # timed iterations against the event-timed window
        "timing_identity": {"sum_phases_ms": float(np.sum(sw) + np.sum(xc) + np.sum(im)), "window_ms": ms,
                            "rel_gap": float((ms - (np.sum(sw) + np.sum(xc) + np.sum(im))) / ms)},
        "final_err": float(errs[-1]) if len(errs) else None,
        "roofline": roof, "clocks": clocks,
        "exchange_used": {rbg.COMM_NONE: "none", rbg.COMM_PEER: "peer", rbg.COMM_NCCL: "nccl"}[comm],
        **({"exchange_fallback": fallback} if fallback else {}),
        **({"replicas_bit_identical": replicas} if replicas is not None else {}),
        # ours per iteration: sweep + IMGS (+ the PEER wait kernel); NCCL's own kernel not counted
        "gpu_launches": (3 if comm == rbg.COMM_PEER else 2) * K,
    }

    # the oracle's sample: the first CPU_SAMPLE_COLS columns of the very bytes the GPU streamed
    host_sample = S[:CPU_SAMPLE_COLS].cpu().numpy() if (rank == 0 and world == 1 and not a.no_cpu) else None

    # ---- end to end through the C ABI with host buffers (pinned), all iterations
    if not a.no_e2e:
        # the host copy needs |S| of pinned RAM per rank on this node: all ranks agree first
        need = S.numel() * S.element_size() * int(os.environ.get("LOCAL_WORLD_SIZE", "1")) * 1.15
        ok = host_mem_available() > need
        if world > 1:
            t = torch.tensor([1 if ok else 0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = bool(t.item())
        if ok:
            host = torch.empty(S.shape, dtype=S.dtype, pin_memory=True)
            host.copy_(S)
            del S
            torch.cuda.empty_cache()
            line["e2e"] = e2e(a, host, w, k_max, W + K, stream, rank, world, M_loc, M_glob, dev, comm)
            del host
        else:
            line["e2e"] = {"value": None, "unit": "it/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                           "note": f"not run: host RAM available {host_mem_available() / 1e9:.0f} GB < "
                                   f"{need / 1e9:.0f} GB needed for pinned host copies of the input"}
    S = None
    torch.cuda.empty_cache()

    # ---- CPU oracle baseline (rank 0, one GPU only): the same k window as the timed
    # region (iterations W..W+K-1), on a bounded column sample (~10-30 s of CPU work)
    if rank == 0 and world == 1 and not a.no_cpu:
        r, wall = cpu_sample(CPU_SAMPLE_COLS, W + K, S=host_sample)
        del host_sample
        t_full = full_iter_seconds(r, W, W + K, CPU_SAMPLE_COLS, M_glob)
        sweep_s = float(np.mean(np.asarray(r.t_iter[W:W + K]) - np.asarray(r.t_imgs[W:W + K])))
        line["cpu_baseline"] = {
            "value": 1.0 / t_full, "unit": "it/s", "cores": oracle_cores(), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sweep_gbs": CPU_SAMPLE_COLS * N * 16 / sweep_s / 1e9,
            "sample": f"CPU oracle (canonical lanes, OpenMP) on the first {CPU_SAMPLE_COLS} of the {M_glob} "
                      f"device columns (same bytes) x {N} rows, iterations {W}..{W + K - 1} ({wall:.1f} s "
                      f"wall); sweep+pivot time scaled by {M_glob}/{CPU_SAMPLE_COLS}, IMGS as measured"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def host_mem_available() -> float:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return float(line.split()[1]) * 1024.0
    except OSError:
        pass
    return 0.0


def e2e(a, host, w, k_max, iters, stream, rank, world, M_loc, M_glob, dev, comm):
    """Same metric through the public API with HOST buffers: H2D of S (pinned host copy)
    inside the timed region (create), all iterations, and the D2H read of pivots, errors
    and basis."""
    import torch
    import torch.distributed as dist
    from paper_1805_06124_b200 import rbg

    S_cols = host.shape
    Sh = host.numpy()
    nccl_id = None
    from paper_1805_06124_b200 import dist as D
    if world > 1:
        dist.barrier()
        if comm == rbg.COMM_NCCL:
            nccl_id = D.nccl_unique_id()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = rbg.Context(Sh, w, 0.0, k_max, stream=stream.cuda_stream, comm=comm, rank=rank, world=world,
                      col_offset=D.partition(M_glob, world, rank)[0], M_global=M_glob, nccl_id=nccl_id)
    if comm == rbg.COMM_PEER:
        D.connect_peers(ctx)
    ctx.step(iters)
    piv = ctx.pivots()
    err = ctx.errors()
    Q = ctx.basis()
    t1 = time.perf_counter()
    wall = D.max_over_ranks(t1 - t0, device=dev)
    ctx.close()
    del Sh
    h2d = S_cols[0] * S_cols[1] * 16
    d2h = piv.nbytes + err.nbytes + Q.nbytes
    return {"value": iters / wall * (M_glob / M_PER_GPU), "unit": "it/s",
            "h2d_bytes_per_step": h2d / iters, "d2h_bytes_per_step": d2h / iters,
            "wall_s": wall, "steps": iters,
            "note": "rbg_create from pinned host S (H2D + NaN scan) + all iterations + D2H of "
                    "pivots/errors/basis, wall clock with device sync"}


def main():
    a = parse()
    if a.strong_cols:
        world = a.gpus
        if a.strong_cols % world:
            raise SystemExit("--strong-cols must be divisible by --gpus")
        a.cols_per_gpu = a.strong_cols // world
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
