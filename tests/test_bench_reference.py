"""The bench's reference arm (the CPU oracle, `bench.py --impl reference`) prints one JSON line
with the contract's keys; under torchrun only rank 0 prints.  Plus the N > 1 bookkeeping of
bench.py's own arm without a GPU (`--dry-run` under torchrun with 8 gloo ranks)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--cols-per-gpu", "3000", "--rows", "1000"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.strip()]


def test_reference_arm_json_contract():
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "it/s" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("reduced") and d["config"]["cols_global"] == 3000
    # at N = 1 every column is run (no extrapolation): the timed region is the measured one
    assert d["extrapolated"] is False and "all 3000 columns" in d["cpu_baseline"]["sample"]
    assert abs(d["timed_region_s"] - d["steps"] * d["ms_per_step"] / 1e3) < 1e-9 * max(1.0, d["timed_region_s"])


def test_reference_arm_nonzero_rank_is_silent():
    assert _run({"RANK": "1"}) == []


def test_default_workload_names_config2_and_config3():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse([])
    assert bench.config_dict(a, 1)["workload"].startswith("config2") and a.cols_per_gpu == 409_600
    a = bench.parse(["--gpus", "8"])
    assert bench.config_dict(a, 8)["workload"].startswith("config3 weak")
    a = bench.parse(["--gpus", "8", "--strong-cols", "1638400"])
    assert a.cols_per_gpu == 204_800 and bench.config_dict(a, 8)["workload"].startswith("config3 strong")


def test_dry_run_eight_ranks_bookkeeping():
    """N = 8 on CPU (gloo): rank 0 alone prints; the contiguous partition covers 3,276,800 columns
    with 409,600 per rank; every rank's e2e host-RAM guard counts LOCAL_WORLD_SIZE = 8 pinned
    copies of its 65.5 GB block (the ranks agree on one outcome); the value is the job's plain
    greedy it/s."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "8",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"), "--gpus", "8",
           "--dry-run"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 8 and d["config"]["cols_global"] == 3_276_800
    assert d["config"]["workload"].startswith("config3 weak") and d["config"]["exchange"] == "peer"
    assert "greedy iterations/s of the whole job" in d["config"]["value_unit"]
    plans = d["plans"]
    assert [p["rank"] for p in plans] == list(range(8))
    off = 0
    for p in plans:
        assert p["col_offset"] == off and p["cols"] == 409_600 and p["cfg"] == 3 and p["local_world"] == 8
        assert p["e2e_guard"]["need_bytes"] == 10_000 * 409_600 * 16 * 8 * 1.15
        off += p["cols"]
    assert off == 3_276_800
    assert d["e2e_runs"] == all(p["e2e_guard"]["run"] for p in plans)


def test_reference_arm_two_ranks_all_columns():
    """Under torchrun with 2 ranks the reference arm runs on rank 0 alone, on all columns of the
    job when they fit host RAM (not extrapolated), with every host core (torchrun workers start
    with OMP_NUM_THREADS=1: the arm sets its thread count explicitly)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29573", os.path.join(ROOT, "bench.py"), "--impl",
           "reference", "--gpus", "2", "--steps", "2", "--warmup", "1", "--cols-per-gpu", "1500", "--rows", "1000"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["extrapolated"] is False
    assert "all 3000 columns" in d["cpu_baseline"]["sample"] and d["cpu_baseline"]["cores"] >= 1
