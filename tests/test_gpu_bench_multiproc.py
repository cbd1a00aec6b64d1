"""bench.py's N > 1 path across real processes (it had never executed).

Two ranks launched by torchrun, each its own process with its own CUDA context, both on cuda:0
(RBG_BENCH_DEVICE=0, gloo process group).  Kernels of different processes must never wait on
each other on one GPU (B200_PROFILING.md: that raised Xid 109), so the exchange runs either as
PEER with a host barrier between every sweep and decision (the sweep's record stores into the
other process's memory and the decision's read of the owner's send slot go through real
cudaIpcOpenMemHandle mappings, the wait kernel finds every tag already released) or through the
process group (EXTERNAL slots, host-staged over gloo).  Checked: rank 0 alone prints the JSON
line; the exchange mode is the one asked for; the replicated IMGS left bit-identical results on
both ranks; and pivots, errors, nu, Q and R equal the canonical-mode CPU oracle on the same bytes
bit for bit (R rows 0..k-2: after rbg_step the sweep with q_{k-1} is still pending).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("comm,port", [("peer-lockstep", 29611), ("host", 29612)])
def test_bench_two_processes_on_one_gpu(orc, tmp_path, comm, port):
    W, K, rows, cols = 3, 12, 1000, 4096
    dump = str(tmp_path / "res")
    args = ["--comm", "peer", "--lockstep"] if comm == "peer-lockstep" else ["--comm", "host"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--pg", "gloo", *args, "--rows", str(rows), "--cols-per-gpu", str(cols),
           "--steps", str(K), "--warmup", str(W), "--no-cpu", "--dump", dump, "--dump-inputs"]
    env = dict(os.environ, RBG_BENCH_DEVICE="0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]                 # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == K and d["value"] > 0
    assert d["exchange_used"] == comm and d["replicas_bit_identical"] is True
    assert d["config"]["cols_global"] == 2 * cols and d["e2e"]["value"] and d["e2e"]["value"] > 0
    # the host barriers / staging between iterations sit outside the per-phase events here
    assert 0.0 <= d["timing_identity"]["rel_gap"] < 1.0

    r = [np.load(f"{dump}.rank{p}.npz") for p in range(2)]
    assert int(r[0]["col_offset"]) == 0 and int(r[1]["col_offset"]) == cols
    for key in ("pivots", "errors", "nu", "Q"):
        np.testing.assert_array_equal(r[0][key], r[1][key])
    S = np.concatenate([r[0]["S"], r[1]["S"]])
    w = r[0]["w"]
    k = W + K
    o = orc.greedy(S, w, 0.0, k, lanes=orc.CANONICAL, max_iters=k)
    assert int(r[0]["k"]) == k == o.k
    np.testing.assert_array_equal(r[0]["pivots"], o.pivots)
    assert (r[0]["pivots"] >= cols).any() and (r[0]["pivots"] < cols).any()   # both ranks own pivots
    np.testing.assert_array_equal(r[0]["errors"], o.errors[:k])
    np.testing.assert_array_equal(r[0]["nu"], o.nu)
    np.testing.assert_array_equal(r[0]["Q"], o.Q)
    R = np.concatenate([r[0]["R"], r[1]["R"]], axis=1)
    np.testing.assert_array_equal(R[:k - 1], o.R[:k - 1])
