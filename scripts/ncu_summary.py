#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list (gpu__time_duration per kernel, share
of the step) and the key metrics of one `--set full` capture.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01/launches.txt
    python scripts/ncu_summary.py full gpurun_out/prof_sweep.ncu-rep > profiles/r01/sweep_full.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second", "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale
        order.append((name, float(d["Metric Value"].replace(",", "")) * scale))
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {path} (cold-cache, serialised; compare shares, not absolutes)")
    print(f"{'launches':>8} {'total_us':>12} {'avg_us':>10} {'share':>7}  kernel")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t:12.1f} {t / c:10.1f} {100 * t / tot:6.1f}%  {n}")
    print("\n# per launch, in order")
    for n, t in order:
        print(f"{t:12.1f} us  {n}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    print(f"# ncu --set full summary: {path}")
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(f"\n## {d.get('Kernel Name', '?')[:120]}  (launch id {d.get('ID')})")
        for k in KEYS:
            if k in d:
                print(f"{k:62s} {u[h.index(k)]:>14s} {d[k]}")
        stalls = [(k, float(d[k])) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and d.get(k, "").replace(".", "").isdigit()]
        tot = sum(s for _, s in stalls) or 1.0
        print("### pc-sampling stall reasons (share of samples)")
        for k, s in sorted(stalls, key=lambda x: -x[1])[:10]:
            if s:
                print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):34s} {100 * s / tot:5.1f}%")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
