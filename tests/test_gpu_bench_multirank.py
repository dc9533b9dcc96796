"""bench.py's N > 1 path (torchrun, one process per rank) on the one GPU this round
has: two ranks share cuda:0 with the gloo backend (NCCL refuses two ranks on one
device).  Covers the ZeroPlan shard-local updates, row-split AdaLomo with its
all-reduces, the fused peer-memory step over CUDA IPC, the end-to-end host-span path on
every rank, and the rank-0 JSON line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_line():
    env = dict(os.environ, MCO_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--layers", "2", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert set(d["per_optimizer"]) == {"adamw", "lion", "adan", "sophia", "lomo", "adalomo"}
    assert d["collectives"]["ms"] > 0 and d["gpu_launches"] > 0
    # e2e over both ranks' host-span calls (max-over-ranks time, whole-job bytes)
    e = d["e2e"]
    assert e["value"] > 0 and set(e["per_optimizer"]) == set(d["per_optimizer"])
    assert e["h2d_bytes_per_step"] == 6 * 2 * 4 * e["params"] == 2 * e["d2h_bytes_per_step"]
