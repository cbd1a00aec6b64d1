"""bench.py's own arm on a small workload (the contract the driver parses): one JSON line with
value, roofline, clocks, e2e and gpu_launches; K timed steps of the real greedy."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_small_workload_json_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--cols-per-gpu", "20480", "--steps", "20", "--warmup", "3",
           "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["steps"] == 20 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["gpu_launches"] == 2 * 20                      # one sweep + one IMGS per timed step
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] and r["achieved"] > 0
    assert abs(d["timing_identity"]["rel_gap"]) < 0.01      # P:946-955 identity within 1 %
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
