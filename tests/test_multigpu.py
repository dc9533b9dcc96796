"""Real multi-GPU runs of the sharded paths (one process per GPU, NCCL), skipped unless
the box has >= 2 GPUs.  Every rank starts from the same parameters with its own
gradients; the result must equal the serial FlatOptimizer step on the rank-summed
gradient (SerialBaseline, tests/serial_ref.hpp:34-70) -- bit for bit where the sum
order is the rank order (peer-memory kernel; any two-rank sum), within one fp32
rounding of the sum otherwise (NCCL's reduction order).

Paths: zero.ZeroShardedOptimizer (torch.distributed RS / AG), zero.NativeZeroOptimizer
(mco_shard_step over the library's NCCL communicator; mco_shard_step_mixed with bf16
replicas), zero.BucketedZeroOptimizer (the bucketed, double-buffered mco_zb step: fp32
replicas and the C4 mixed layout), zero.PeerShardedOptimizer (one kernel over NVLink
peer memory); the C3 / C5 paths of tests/test_gpu_dp_processes.py over NCCL
(zero.RowShardedAdaLomo with its statistic all-reduces and the clip, zero.ZeroShardedLomo
and the bf16 owned-shard LOMO with the global clip); and bench.py under torchrun with
NCCL (the rank count NCCL reports checked against --gpus)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
needs_multi = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
WORLD = min(NGPU, 4)
P = 1000003  # not divisible by 2, 3 or 4: uneven ZeroPlan parts, odd shard offsets
STEPS = 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _grad(rank, t):
    return O.synth(P, 41, 1, rank, t, 0, -7, 10, False)


def _worker(rank, world, port, q):
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    import torch.distributed as dist

    from paper_2312_00407_b200 import zero
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    out = {}
    try:
        cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
        cfg.weight_decay = 0.01
        p0 = torch.from_numpy(O.synth(P, 41, 0, 0, 0, 0, -6, 0, False)).cuda()

        z = zero.ZeroShardedOptimizer(cfg, P)
        p = p0.clone()
        for t in range(1, STEPS + 1):
            z.step(p, torch.from_numpy(_grad(rank, t)).cuda(), 1e-3)
        out["zero"] = p.cpu().numpy()

        comm = zero.NcclComm()
        nz = zero.NativeZeroOptimizer(cfg, P, comm)
        p = p0.clone()
        for t in range(1, STEPS + 1):
            nz.step(p, torch.from_numpy(_grad(rank, t)).cuda(), 1e-3)
        torch.cuda.synchronize()
        comm.check()
        out["native"] = p.cpu().numpy()

        nm = zero.NativeZeroOptimizer(cfg, P, comm, mixed=True, master_init=p0)
        rep = p0.bfloat16()
        for t in range(1, STEPS + 1):
            nm.step(rep, torch.from_numpy(_grad(rank, t)).cuda(), 1e-3)
        torch.cuda.synchronize()
        out["native_mixed"] = rep.float().cpu().numpy()

        zb = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=100000)
        p = p0.clone()
        for t in range(1, STEPS + 1):
            zb.step(p, torch.from_numpy(_grad(rank, t)).cuda(), 1e-3)
        torch.cuda.synchronize()
        comm.check()
        out["bucketed"] = p.cpu().numpy()

        zm = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=100000,
                                        replica_dtype=torch.bfloat16)
        zm.load_master(p0)
        rep = torch.zeros(P, dtype=torch.bfloat16, device="cuda")
        for t in range(1, STEPS + 1):
            zm.step(rep, torch.from_numpy(_grad(rank, t)).cuda(), 1e-3)
        torch.cuda.synchronize()
        out["bucketed_mixed"] = rep.float().cpu().numpy()

        ps = zero.PeerShardedOptimizer(cfg, P)
        ps.params.copy_(p0)
        for t in range(1, STEPS + 1):
            ps.grads.copy_(torch.from_numpy(_grad(rank, t)).cuda())
            torch.cuda.synchronize()
            ps.step(1e-3)
        torch.cuda.synchronize()
        out["peer"] = ps.params.cpu().numpy()
        dist.barrier()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    if NGPU < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _serial():
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
    cfg.weight_decay = 0.01
    p = O.synth(P, 41, 0, 0, 0, 0, -6, 0, False)
    orc = O.OracleFlat(cfg, P, np.float32)
    for t in range(1, STEPS + 1):
        g = _grad(0, t)
        for r in range(1, WORLD):
            g = g + _grad(r, t)  # rank order, fp32
        orc.step(p, g, 1e-3)
    return p


@needs_multi
@pytest.mark.parametrize("path", ["zero", "native", "peer", "native_mixed", "bucketed",
                                  "bucketed_mixed"])
def test_sharded_paths_equal_serial(results, path):
    want = _serial()
    if path.endswith("_mixed"):  # bf16 replicas of the fp32 master (RNE)
        want = torch.from_numpy(want).bfloat16().float().numpy()
    for r in range(WORLD):
        got = results[r][path]
        assert np.array_equal(got, results[0][path])  # replicas agree bit for bit
        if path == "peer" or WORLD == 2:
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        else:  # NCCL sums in its own order: the gradient may differ by one rounding
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-9)


@needs_multi
@pytest.mark.parametrize("clip", [1e-3, None])
def test_row_sharded_adalomo_nccl_matches_reference(clip):
    from test_gpu_dp_processes import check_row_sharded_adalomo
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    check_row_sharded_adalomo(WORLD, clip, "nccl")


@needs_multi
def test_zero_sharded_lomo_nccl_matches_reference():
    from test_gpu_dp_processes import check_zero_sharded_lomo
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    check_zero_sharded_lomo(WORLD, "nccl")


@needs_multi
def test_sharded_lomo_bf16_nccl_matches_restatement():
    from test_gpu_dp_processes import check_sharded_lomo_bf16
    check_sharded_lomo_bf16(WORLD, "nccl")


@needs_multi
def test_bench_under_torchrun_nccl():
    """bench.py --gpus N under torchrun: one line, n_gpus = N = the rank count NCCL's own
    init log reports, the value = 6 P / the summed whole-DP-step times, every kind with
    its shard-local time and NVLink bytes."""
    import re

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={WORLD}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), "bench.py", "--gpus", str(WORLD), "--steps", "2", "--warmup", "1",
           "--layers", "2", "--no-e2e", "--no-cpu-baseline", "--repeats", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == WORLD and d["value"] > 0 and d["scaling"] == "strong"
    assert d["collectives"]["backend"] == "nccl"
    assert d["collectives"]["nccl_allgather_busbw_gbs"] > 0
    nr = {int(m) for m in re.findall(r"nRanks (\d+)", r.stderr)}
    assert nr == {WORLD}, sorted(nr)  # NCCL_DEBUG=INFO (bench.py sets it for N > 1)
    P = d["config"]["params"]
    for k, e in d["per_optimizer"].items():
        assert e["shard_local"]["ms"] > 0 and e["nvlink"]["bytes_per_rank_per_direction"] > 0, k
    total = sum(e["ms"] for e in d["per_optimizer"].values())
    assert abs(d["value"] - len(d["per_optimizer"]) * P / (total * 1e-3)) / d["value"] < 1e-4
