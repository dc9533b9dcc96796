"""bench.py's N > 1 path on the one GPU a test box has: `python bench.py --gpus 2`
re-launches itself with two ranks (torch.distributed.run) that share cuda:0 over gloo
(NCCL refuses two ranks on one device).  Covers the whole data-parallel step per
optimizer (gradient reduce-scatter -> update -> parameter all-gather; LOMO's clip
all-reduce; row-split AdaLomo with its rank-major reduce-scatter / all-gather and two
statistic all-reduces), the shard-local figure beside it, the end-to-end host-span path
on every rank, and the single rank-0 JSON line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_line():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["MCO_BENCH_BACKEND"] = "gloo"
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--layers", "2", "--no-cpu-baseline", "--repeats", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    kinds = {"adamw", "lion", "adan", "sophia", "lomo", "adalomo"}
    assert set(d["per_optimizer"]) == kinds
    P = d["config"]["params"]
    for k, e in d["per_optimizer"].items():
        assert e["shard_local"]["ms"] > 0, k
        assert e["nvlink"]["bytes_per_rank_per_direction"] >= P * 4, k  # RS + AG, fp32
        # value = 6 P / sum of the whole-step times
    total = sum(e["ms"] for e in d["per_optimizer"].values())
    assert abs(d["value"] - 6 * P / (total * 1e-3)) / d["value"] < 1e-5  # ms are rounded to 4 decimals
    assert d["gpu_launches"] > 0 and d["collectives"]["backend"] == "gloo"
    # e2e over both ranks' host-span calls (max-over-ranks time, whole-job bytes)
    e = d["e2e"]
    assert e["value"] > 0 and set(e["per_optimizer"]) == kinds
    # 8 B/param up (p, g) per optimizer (LOMO's clip pass keeps g resident); 4 B down
    assert e["h2d_bytes_per_step"] == 6 * 8 * e["params"]
    assert e["d2h_bytes_per_step"] == 6 * 4 * e["params"]
