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

``value`` is the greedy's iteration rate (BASELINE.json's "greedy iterations/s"): one
iteration of the whole job advances the basis of the whole M_global-column matrix by one
vector, so at N GPUs it is the job's rate, and weak scaling keeps it flat when every GPU
holds 409,600 columns; ``colit_per_s`` (column-iterations/s = it/s x M_global) is the work
throughput.  The JSON line also carries the fused sweep's roofline (HBM bytes per launch /
event-timed duration, against MEASURED_PEAKS.json), the CPU oracle baseline on all columns
for a bounded number of iterations, an end-to-end number through the C ABI with host
buffers, and the SM clocks seen during the timed region.

Multi-process modes for a box with fewer GPUs than ranks (tests; never the driver's run):
``--pg gloo`` + ``RBG_BENCH_DEVICE=0`` put every rank on one GPU; there the exchange must not
have kernels of different processes wait for each other (B200_PROFILING.md: Xid 109), so
``--comm peer --lockstep`` separates each iteration's sweep and decision by host barriers
(real CUDA-IPC stores/loads, no waiting kernel ever spins), and ``--comm host`` moves the
slots through the process group (EXTERNAL exchange).  ``--dry-run`` prints every rank's plan
(partition, e2e host-RAM guard) without a GPU.
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
SPEC_HBM_GBS = 8000.0          # B200 datasheet HBM3e bandwidth (context)
# measured read-only ceiling of the sweep's own access pattern on this pool's B200s (one warp
# per 160 KB column, 16-byte loads, columns dealt dynamically from a grid-wide counter, best
# of the T/U/occupancy variants): scripts/hbm_probe2.cu, profiles/r01/hbm_probe2.txt
READ_STREAM_GBS = 7465.3
CPU_MAX_ITERS = 25             # oracle iterations timed on the host (about 20 s on 16 cores)


def parse(argv=None):
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
    p.add_argument("--graph-batch", type=int, default=0,
                   help="time CUDA-graph batches of this many iterations (no per-phase events; the "
                        "roofline then charges the whole step to the sweep)")
    p.add_argument("--ortho", default="mgs", choices=["mgs", "cgs"],
                   help="IMGS variant: the paper's MGSCI (default) or Hoffmann CGSCI")
    p.add_argument("--residual", default="recurrence", choices=["recurrence", "explicit"],
                   help="column residuals: the paper's recurrence (default) or Algorithm 2 updates")
    p.add_argument("--comm", default="peer", choices=["peer", "nccl", "host"],
                   help="N > 1 exchange: records/pivot column over NVLink inside the kernels (default), "
                        "one ncclAllGather per iteration, or the slots moved through the process group")
    p.add_argument("--lockstep", action="store_true",
                   help="PEER: host barrier between every sweep and decision (ranks sharing a GPU)")
    p.add_argument("--pg", default="nccl", choices=["nccl", "gloo"],
                   help="torch.distributed backend (gloo: ranks sharing a GPU, CPU dry runs)")
    p.add_argument("--dump", default="",
                   help="write every rank's results (and its S block if --dump-inputs) to DUMP.rank<r>.npz")
    p.add_argument("--dump-inputs", action="store_true")
    p.add_argument("--dry-run", action="store_true",
                   help="no GPU: print every rank's partition / e2e guard / config (gloo)")
    a = p.parse_args(argv)
    if a.strong_cols:
        if a.strong_cols % a.gpus:
            raise SystemExit("--strong-cols must be divisible by --gpus")
        a.cols_per_gpu = a.strong_cols // a.gpus
    return a


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


def host_mem_available() -> float:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return float(line.split()[1]) * 1024.0
    except OSError:
        pass
    return 0.0


def env_ranks():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("LOCAL_WORLD_SIZE", "1")))


def plan(a, rank: int, world: int) -> dict:
    """This rank's share of the workload: contiguous column blocks (dist.partition)."""
    from paper_1805_06124_b200 import dist as D
    M_glob = a.cols_per_gpu * world
    off, m_loc = D.partition(M_glob, world, rank)
    return {"rank": rank, "world": world, "rows": a.rows, "col_offset": off, "cols": m_loc,
            "cols_global": M_glob, "cfg": 2 if world == 1 else 3,
            "k_max": max(K_MAX, a.warmup + a.steps), "s_bytes": a.rows * m_loc * 16}


def e2e_guard(s_bytes: int, local_world: int, available: float) -> dict:
    """The e2e leg pins a host copy of every local rank's S: run it only if the node's free
    RAM covers all of them with 15 % headroom (all ranks agree on the outcome)."""
    need = s_bytes * local_world * 1.15
    return {"need_bytes": need, "available_bytes": available, "run": available > need}


def config_dict(a, world):
    if getattr(a, "strong_cols", 0):
        wl = f"config3 strong: 10,000 x {a.strong_cols} over {world} GPUs ({a.cols_per_gpu} per GPU), k_max 300"
    elif world == 1:
        wl = "config2: complex fp64 chirp snapshots 10,000 x 409,600 (65.5 GB), k_max 300"
    else:
        wl = f"config3 weak: 10,000 x 409,600 per GPU x {world} GPUs, k_max 300"
    if a.rows != N_ROWS or (a.cols_per_gpu != M_PER_GPU and not a.strong_cols):
        wl = f"reduced: {a.rows} x {a.cols_per_gpu} per GPU x {world} GPUs (not a BASELINE config), k_max {max(K_MAX, a.warmup + a.steps)}"
    exch = "none"
    if world > 1:
        exch = a.comm + ("-lockstep" if a.comm == "peer" and a.lockstep else "")
    return {"workload": wl,
            "rows": a.rows, "cols_per_gpu": a.cols_per_gpu, "cols_global": a.cols_per_gpu * world,
            "k_window": [a.warmup, a.warmup + a.steps], "parallelism": f"column-sharded x{world}",
            "l2": "inputs (65.5 GB/GPU) >> 126 MB L2; no flush",
            "ortho": getattr(a, "ortho", "mgs"), "residual": getattr(a, "residual", "recurrence"),
            "exchange": exch, "process_group": a.pg,
            "value_unit": "greedy iterations/s of the whole job (basis vectors per second); "
                          "colit_per_s = it/s x cols_global"}


# ----------------------------------------------------------------------------- reference arm

def run_reference(a):
    """The CPU oracle (oracle/, as it stands) on the box's host cores, on this arm's workload:
    all M_global columns (generated on the host with every core) when they fit host RAM (always
    at N = 1), iterations 0..W+K-1 actually run and iterations W..W+K-1 timed.  Otherwise (e.g.
    N x 65.5 GB at N = 4, 8) one GPU's 409,600 columns are timed and the column sweep scaled by
    M_global / 409,600."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1805_06124_b200 import inputs
    world = a.gpus
    W, K = a.warmup, a.steps
    M_glob = a.cols_per_gpu * world
    # all columns when the job fits host RAM (S plus the oracle's R and headroom), else one GPU's
    need = M_glob * a.rows * 16 + (W + K) * M_glob * 16
    cols = M_glob if need * 1.1 < host_mem_available() or world == 1 else a.cols_per_gpu
    cfg = 2 if world == 1 else 3
    t0 = time.perf_counter()
    t = inputs.chirp_grid(a.rows)
    w = inputs.simpson_weights(a.rows)
    q, chi, psi = inputs.chirp_params(M_glob, cfg, spin=True)
    S = inputs.chirp_columns_host(t, w, q[:cols], chi[:cols], psi[:cols], spin=True)
    t_gen = time.perf_counter() - t0
    # all host cores explicitly: torchrun starts its workers with OMP_NUM_THREADS=1
    r = O.greedy(S, w, 0.0, W + K, lanes=O.CANONICAL, max_iters=W + K, threads=oracle_cores())
    if r.k != W + K:
        raise SystemExit(f"oracle stopped early ({r.stop} at k={r.k})")
    t_it = np.asarray(r.t_iter[W:W + K])
    t_im = np.asarray(r.t_imgs[W:W + K])
    scale = M_glob / cols
    per = (t_it - t_im) * scale + t_im              # scale = 1 at N = 1: measured as is
    val = K / float(np.sum(per))
    cores = oracle_cores()
    sample = (f"CPU oracle (canonical lanes, OpenMP) on all {cols} columns x {a.rows} rows, iterations "
              f"0..{W + K - 1} run, {W}..{W + K - 1} timed (input generated on the host in {t_gen:.1f} s)"
              if scale == 1 else
              f"CPU oracle on one GPU's {cols} of {M_glob} columns x {a.rows} rows, iterations {W}..{W + K - 1}; "
              f"column sweep time x {scale:g} (the whole job does not fit host RAM), IMGS as measured")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "it/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": float(np.mean(per)) * 1e3, "higher_is_better": True,
        "scaling": "strong" if a.strong_cols else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (host-generated chirps, BASELINE.json config 2/3 recipe)",
        "config": config_dict(a, world), "colit_per_s": val * M_glob,
        "timed_region_s": float(np.sum(t_it)), "extrapolated": scale != 1,
        "cpu_baseline": {"value": val, "unit": "it/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sweep_gbs": cols * a.rows * 16 / float(np.mean(t_it - t_im)) / 1e9, "sample": sample},
        "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm

class Driver:
    """Enqueues greedy iterations on a context in the bench's exchange mode."""

    def __init__(self, ctx, mode: str, stream, world: int):
        self.ctx, self.mode, self.stream, self.world = ctx, mode, stream, world

    def step(self, n: int):
        import torch.distributed as dist
        from paper_1805_06124_b200 import dist as D
        if self.mode == "lockstep":
            # PEER with a host barrier between every sweep (which stores its record into every
            # rank's memory over CUDA IPC) and every decision (whose wait kernel then finds all
            # tags released): no kernel ever waits for another process's kernel
            for _ in range(n):
                self.ctx.iter_local()
                self.stream.synchronize()
                dist.barrier()
                self.ctx.iter_finish()
                self.stream.synchronize()
                dist.barrier()
        elif self.mode == "host":
            for _ in range(n):
                self.ctx.iter_local()
                D.exchange_slots(self.ctx, stream=self.stream)
                self.ctx.iter_finish()
        else:
            self.ctx.step(n)


def replica_hash(ctx) -> str:
    """sha256 of the replicated results (pivots, errors, basis) of a sharded context."""
    import hashlib
    hsh = hashlib.sha256()
    for arr in (ctx.pivots(), ctx.errors(), ctx.basis()):
        hsh.update(np.ascontiguousarray(arr).tobytes())
    return hsh.hexdigest()


def run_dry(a):
    """--dry-run: every rank's plan and e2e guard, gathered to rank 0 (gloo, no GPU)."""
    import torch.distributed as dist
    rank, world, local, local_world = env_ranks()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
    from paper_1805_06124_b200 import dist as D
    pl = plan(a, rank, world)
    pl["local_rank"], pl["local_world"] = local, local_world
    pl["e2e_guard"] = e2e_guard(pl["s_bytes"], local_world, host_mem_available())
    plans = D.all_gather_bytes(pl) if world > 1 else [pl]
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "config": config_dict(a, world),
                          "e2e_runs": all(p["e2e_guard"]["run"] for p in plans), "plans": plans}), flush=True)
    return 0


def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_1805_06124_b200 import dist as D
    from paper_1805_06124_b200 import inputs
    from paper_1805_06124_b200 import rbg

    rank, world, local, local_world = env_ranks()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    dev_idx = int(os.environ.get("RBG_BENCH_DEVICE", local))
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if world > 1:
        if a.pg == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    W, K = a.warmup, a.steps
    if W < 3:
        raise SystemExit("--warmup must be >= 3")
    pl = plan(a, rank, world)
    N, M_loc, M_glob, off, k_max = pl["rows"], pl["cols"], pl["cols_global"], pl["col_offset"], pl["k_max"]

    # ---- synthetic input, generated on the device
    t_grid = inputs.chirp_grid(N)
    w = inputs.simpson_weights(N)
    q, chi, psi = inputs.chirp_params(M_glob, pl["cfg"], spin=True)
    sl = slice(off, off + M_loc)
    S = torch.empty((M_loc, N), dtype=torch.complex128, device=dev)
    rbg.gen_chirp(S, t_grid, w, q[sl], chi[sl], psi[sl], spin=True)

    stream = torch.cuda.Stream(dev)                 # the library enqueues on this stream
    torch.cuda.set_stream(stream)

    mode = "plain"
    if world > 1 and a.comm == "peer" and a.lockstep:
        mode = "lockstep"
    elif world > 1 and a.comm == "host":
        mode = "host"

    def make_ctx(comm, timing=True):
        nccl_id = D.nccl_unique_id() if comm == rbg.COMM_NCCL else None
        ctx = rbg.Context(S, w, 0.0, k_max, stream=stream.cuda_stream, comm=comm, rank=rank,
                          world=world, col_offset=off, M_global=M_glob, nccl_id=nccl_id, ortho=a.ortho,
                          residual=a.residual, peer_timeout_ms=20000)
        if comm == rbg.COMM_PEER:
            D.connect_peers(ctx)
        ctx.set_timing(timing)
        if a.graph_batch:
            ctx.set_graph_batch(a.graph_batch)
        drv = Driver(ctx, mode, stream, world)
        drv.step(W)                                  # warm-up: sweep 0 + W iterations
        torch.cuda.synchronize()
        return ctx, drv

    comm = rbg.COMM_NONE
    if world > 1:
        comm = {"peer": rbg.COMM_PEER, "nccl": rbg.COMM_NCCL, "host": rbg.COMM_EXTERNAL}[a.comm]
    timing = not a.graph_batch
    fallback = None
    if comm == rbg.COMM_PEER and mode == "plain":
        # the PEER exchange needs CUDA IPC between the ranks' processes: if any rank cannot map
        # its peers or the warm-up timed out, every rank falls back to the NCCL exchange
        # -- and so does every rank if the replicated results already differ after the warm-up
        # (the first free-running PEER run on a multi-GPU box must not corrupt the timed record)
        ok, ctx, same = True, None, True
        try:
            ctx, drv = make_ctx(comm, timing)
            ok = ctx.info()[2] != "PEER_TIMEOUT"
        except rbg.RbgError as e:
            ok, fallback = False, str(e)
        ok = min(D.all_gather_bytes(1 if ok else 0)) == 1
        if ok:
            same = len(set(D.all_gather_bytes(replica_hash(ctx)))) == 1
        if not ok or not same:
            if ctx is not None:
                ctx.close()
            fallback = fallback or ("PEER warm-up failed on some rank" if not ok else
                                    "replicas differ after the PEER warm-up")
            comm = rbg.COMM_NCCL
            ctx, drv = make_ctx(comm, timing)
    else:
        ctx, drv = make_ctx(comm, timing)

    # ---- exactly K timed iterations
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev_idx)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    drv.step(K)
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
    errs = ctx.errors()
    gpu_piv, gpu_err = ctx.pivots(), errs
    replicas = None
    if world > 1:
        # the replicated IMGS must leave bit-identical pivots / errors / basis on every rank
        # (SURVEY §5 integrity check): compare a hash of their bits across the ranks
        replicas = len(set(D.all_gather_bytes(replica_hash(ctx)))) == 1
    if a.dump:
        res = ctx.result()
        extra = {"S": S.cpu().numpy(), "w": w} if a.dump_inputs else {}
        np.savez(f"{a.dump}.rank{rank}.npz", k=res.k, pivots=res.pivots, errors=res.errors, nu=res.nu,
                 Q=res.Q, R=res.R, r2=res.r2, col_offset=off, cols_global=M_glob, **extra)

    it_s = K / (ms / 1e3)
    bytes_sweep = N * M_loc * 16 + M_loc * (8 + 8 + 16)      # DESIGN.md "Roofline" per launch
    if a.residual == "explicit":
        bytes_sweep += 2 * N * M_loc * 16                     # + re-read and write-back of V
    pk = peaks()
    peak = pk.get("hbm_gbs") or 6650.0
    roof = {"kernel": "k_sweep_dyn (fused coefficient sweep + r2 update + maxloc, dynamically scheduled columns)",
            "bound": "hbm", "peak": peak, "unit": "GB/s",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if pk.get("hbm_gbs") else "fallback 6.65 TB/s",
            "traffic": ncu_traffic(), "algorithmic_bytes_per_launch": bytes_sweep,
            "read_stream_ceiling_gbs": READ_STREAM_GBS}
    phases = None
    if timing:
        sweep_ms, xchg_ms, imgs_ms = ctx.timings(W + K)
        # iteration t's sweep uses q_{t-1}: timed iterations W..W+K-1 -> sweeps W-1..W+K-2
        sw = sweep_ms[W - 1:W + K - 1]
        im = imgs_ms[W:W + K]
        xc = xchg_ms[W:W + K]
        sweep_avg_s = float(np.mean(sw)) / 1e3
        achieved = bytes_sweep / sweep_avg_s / 1e9
        roof.update({"achieved": achieved, "frac": achieved / peak, "sweep_ms_avg": sweep_avg_s * 1e3,
                     # SURVEY 8(d) quotes the median sweep over iterations k >= 3
                     "sweep_ms_median": float(np.median(sw)),
                     "achieved_at_median_gbs": bytes_sweep / (float(np.median(sw)) / 1e3) / 1e9,
                     "share_of_step": float(np.sum(sw) / ms),
                     # the same bandwidth against the datasheet figure and the
                     # measured read-only ceiling of the same access pattern
                     "frac_of_spec_8tbs": achieved / SPEC_HBM_GBS,
                     "frac_of_read_stream_ceiling": achieved / READ_STREAM_GBS})
        phases = {"phase_ms_avg": {"sweep": float(np.mean(sw)), "xchg": float(np.mean(xc)), "imgs": float(np.mean(im))},
                  # the paper's identity T_j = T_pivot + C_j + T_IMGS, summed
                  # over the timed iterations against the event-timed window
                  "timing_identity": {"sum_phases_ms": float(np.sum(sw) + np.sum(xc) + np.sum(im)), "window_ms": ms,
                                      "rel_gap": float((ms - (np.sum(sw) + np.sum(xc) + np.sum(im))) / ms)}}
    else:
        # graph batches carry no per-phase events: the whole step is charged to the sweep (a
        # lower bound on its bandwidth)
        achieved = bytes_sweep / (ms / K / 1e3) / 1e9
        roof.update({"achieved": achieved, "frac": achieved / peak, "achieved_basis": "whole step (graph batches)",
                     "frac_of_spec_8tbs": achieved / SPEC_HBM_GBS,
                     "frac_of_read_stream_ceiling": achieved / READ_STREAM_GBS})
    per_iter = {"peer": 3, "nccl": 2, "host": 2}.get(a.comm, 2) if world > 1 else 2
    line = {
        "metric": METRIC, "value": it_s, "unit": "it/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "strong" if a.strong_cols else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (device-generated chirps, BASELINE.json config 2/3 recipe)",
        "config": config_dict(a, world), "iters_per_s": it_s, "colit_per_s": it_s * M_glob,
        "hbm_gbs_per_gpu": achieved, "hbm_gbs_total": achieved * world,
        **(phases or {}),
        "launch": f"graph batches of {a.graph_batch}" if a.graph_batch else "plain launches + per-phase CUDA events",
        "final_err": float(errs[-1]) if len(errs) else None,
        "roofline": roof, "clocks": clocks,
        "exchange_used": ({rbg.COMM_NONE: "none", rbg.COMM_PEER: "peer", rbg.COMM_NCCL: "nccl",
                           rbg.COMM_EXTERNAL: "host"}[comm] + ("-lockstep" if mode == "lockstep" else "")),
        **({"exchange_fallback": fallback} if fallback else {}),
        **({"replicas_bit_identical": replicas} if replicas is not None else {}),
        # ours per iteration: sweep + IMGS (+ the PEER wait kernel); NCCL's own kernel not counted
        "gpu_launches": (3 if comm == rbg.COMM_PEER else 2) * K if world > 1 else per_iter * K,
    }
    ctx.close()

    # ---- end to end through the C ABI with host buffers (pinned), all iterations; then the
    # CPU oracle on the same host bytes (rank 0, one GPU)
    host = None
    guard = e2e_guard(pl["s_bytes"], local_world, host_mem_available())
    ok = guard["run"]
    if world > 1:
        ok = min(D.all_gather_bytes(1 if ok else 0)) == 1
    if not a.no_e2e and ok:
        host = torch.empty(S.shape, dtype=S.dtype, pin_memory=True)
        host.copy_(S)
    elif not a.no_e2e:
        line["e2e"] = {"value": None, "unit": "it/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                       "note": f"not run: host RAM available {guard['available_bytes'] / 1e9:.0f} GB < "
                               f"{guard['need_bytes'] / 1e9:.0f} GB needed for pinned host copies of the input"}
    if host is None and rank == 0 and world == 1 and not a.no_cpu:
        host = S.cpu()                                # pageable copy for the oracle only
    del S
    torch.cuda.empty_cache()
    if not a.no_e2e and ok:
        line["e2e"] = e2e(a, host, w, k_max, W + K, stream, rank, world, M_loc, M_glob, dev, comm, mode)

    # ---- CPU oracle baseline (rank 0, one GPU only): all columns of the very bytes the GPU
    # streamed, iterations 0..min(W+K, 25)-1 (about 20 s of CPU work on 16 cores)
    if rank == 0 and world == 1 and not a.no_cpu:
        from oracle import oracle as O
        n_it = min(W + K, CPU_MAX_ITERS)
        lo = min(W, n_it - 1)
        Sh = host.numpy()
        t0 = time.perf_counter()
        r = O.greedy(Sh, w, 0.0, n_it, lanes=O.CANONICAL, max_iters=n_it, threads=oracle_cores())
        wall = time.perf_counter() - t0
        t_it = np.asarray(r.t_iter[lo:n_it])
        t_im = np.asarray(r.t_imgs[lo:n_it])
        line["cpu_baseline"] = {
            "value": len(t_it) / float(np.sum(t_it)), "unit": "it/s", "cores": oracle_cores(), "kind": "oracle",
            "cpu_model": cpu_model(), "sweep_gbs": M_loc * N * 16 / float(np.mean(t_it - t_im)) / 1e9,
            "sample": f"CPU oracle (canonical lanes, OpenMP) on all {M_loc} device columns (same bytes) x {N} "
                      f"rows: sweep 0 + iterations 0..{n_it - 1} run ({wall:.1f} s wall), iterations "
                      f"{lo}..{n_it - 1} timed",
            # the same bytes, the same canonical arithmetic: the first pivots agree bit for bit
            "pivots_match_gpu": bool(np.array_equal(r.pivots, gpu_piv[:n_it])),
            "errors_match_gpu": bool(np.array_equal(r.errors[:n_it], gpu_err[:n_it]))}
    del host
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def e2e(a, host, w, k_max, iters, stream, rank, world, M_loc, M_glob, dev, comm, mode):
    """Same metric through the public API with HOST buffers: H2D of S (pinned host copy)
    inside the timed region (create), all iterations, and the D2H read of pivots, errors
    and basis."""
    import torch
    import torch.distributed as dist
    from paper_1805_06124_b200 import dist as D
    from paper_1805_06124_b200 import rbg

    S_cols = host.shape
    Sh = host.numpy()
    nccl_id = None
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
    t_create = time.perf_counter()
    Driver(ctx, mode, stream, world).step(iters)
    piv = ctx.pivots()                                # synchronises: the iterations are done
    t_iter = time.perf_counter()
    err = ctx.errors()
    Q = ctx.basis()
    t1 = time.perf_counter()
    wall = D.max_over_ranks(t1 - t0, device=dev)
    ctx.close()
    h2d = S_cols[0] * S_cols[1] * 16
    d2h = piv.nbytes + err.nbytes + Q.nbytes
    return {"value": iters / wall, "unit": "it/s",
            "h2d_bytes_per_step": h2d / iters, "d2h_bytes_per_step": d2h / iters,
            "wall_s": wall, "steps": iters,
            # this rank's split of the wall time: the create (65.5 GB over PCIe at ~55 GB/s + the
            # NaN scan) is the floor of this number over a short window
            "split_s": {"create_h2d": t_create - t0, "iterations": t_iter - t_create, "readback": t1 - t_iter},
            "note": "rbg_create from pinned host S (H2D + NaN scan) + all iterations + D2H of "
                    "pivots/errors/basis, wall clock with device sync"}


def main():
    a = parse()
    if a.dry_run:
        return run_dry(a)
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
