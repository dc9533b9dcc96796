"""Multi-process parity of the sharded C3 / C5 paths on the one GPU a test
box has: N OS processes share cuda:0 over a gloo process group (NCCL refuses two ranks
on one device), each holding its own local gradients, and the result is checked
against the compiled reference on the rank-summed gradient.  tests/test_multigpu.py
runs the same checks over NCCL with one GPU per rank (check_* with backend "nccl").

* C3: zero.RowShardedAdaLomo.step_dp -- every matrix split by rows (uneven row counts
  included), replicated 1-D tensors, the global grad-norm clip; reduce-scatter of the
  rank-major gradients, the column-statistic / Σg² all-reduce (optim.cpp:241-249 across
  ranks), the Σu² all-reduce, all-gather.  Oracle: the reference's clip rule
  (optim.cpp:302-303) scaling the summed gradient, then the reference
  AdaLomoState::apply (the reference's own TP variant, parallel.cpp:334, keeps local
  statistics and is not used).
* C5: zero.ZeroShardedLomo (reduce-scatter -> Σg² all-reduce -> clipped update ->
  all-gather, fp32) vs the reference's two-pass lomo_fused_backward_step
  (optim.cpp:284-318) on the summed gradient; and the bf16 owned-shard form
  (zero.sharded_lomo_step on bf16 parameters / gradients) vs the bf16 restatement with
  the global clip scale -- the reference forbids the clip in parallel runs
  (parallel.cpp:335-337).
"""
import os
import socket
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")

ADA_SHAPES = [(40, 24), (8,), (37, 16), (24, 40), (5,), (9, 8)]
ADA_STEPS, ADA_LR = 2, 5e-3
LOMO_P, LOMO_STEPS, LOMO_LR = 100003, 2, 1e-2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ada_grads(rank, t):
    return np.concatenate(O.registry_grads(ADA_SHAPES, 300 + rank, t, np.float32))


def _lomo_grad(rank, t, n=LOMO_P):
    return O.synth(n, 61, 1, rank, t, 0, -7, 10, False)


def _worker(what, rank, world, port, arg, q, backend="gloo"):
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2312_00407_b200 import optim, zero
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if backend == "nccl":  # one GPU per rank (tests/test_multigpu.py)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
    else:  # ranks sharing cuda:0
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
    try:
        if what == "ada":
            cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
            rs = zero.RowShardedAdaLomo(cfg, ADA_SHAPES, grad_clip=arg)
            p = torch.from_numpy(np.concatenate(
                O.registry_params(ADA_SHAPES, 77, np.float32))).cuda()
            rm_p = rs.to_rank_major(p)
            for t in range(1, ADA_STEPS + 1):
                g = torch.from_numpy(_ada_grads(rank, t)).cuda()
                rs.step_dp(rm_p, rs.to_rank_major(g), ADA_LR)
            rs.from_rank_major(rm_p, p)
            torch.cuda.synchronize()
            q.put((rank, p.cpu().numpy()))
        elif what == "lomo32":
            zl = zero.ZeroShardedLomo(LOMO_P, clip=arg)
            p = torch.from_numpy(O.synth(LOMO_P, 61, 0, 0, 0, 0, -6, 0, False)).cuda()
            for t in range(1, LOMO_STEPS + 1):
                zl.step(p, torch.from_numpy(_lomo_grad(rank, t)).cuda(), LOMO_LR)
            torch.cuda.synchronize()
            q.put((rank, p.cpu().numpy()))
        else:  # "lomo_bf16": the C5 layout -- owned bf16 shards, gradients already reduced
            plan = zero.ZeroPlan.make(LOMO_P, world)
            lo, hi = plan.owned_range(rank)
            p0 = O.f32_to_bf16(O.synth(LOMO_P, 62, 0, 0, 0, 0, -6, 0, False))[lo:hi]
            p = torch.from_numpy(p0.view(np.int16).copy()).cuda().view(torch.bfloat16)
            for t in range(1, LOMO_STEPS + 1):
                g = O.f32_to_bf16(O.synth(LOMO_P, 62, 1, 0, t, 0, -7, 10, False))[lo:hi]
                tg = torch.from_numpy(g.view(np.int16).copy()).cuda().view(torch.bfloat16)
                zero.sharded_lomo_step(p, tg, LOMO_LR, arg)
            torch.cuda.synchronize()
            q.put((rank, p.view(torch.int16).cpu().numpy().view(np.uint16)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(what, world, arg, backend="gloo"):
    import torch.multiprocessing as mp

    port = _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(what, r, world, port, arg, q, backend))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@needs_ref
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("clip", [1e-3, None])
def test_row_sharded_adalomo_processes_match_reference(world, clip):
    check_row_sharded_adalomo(world, clip, "gloo")


def check_row_sharded_adalomo(world, clip, backend):
    res = _run("ada", world, clip, backend)
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ps = O.registry_params(ADA_SHAPES, 77, np.float64)
    p0 = [x.copy() for x in ps]
    r = O.RefAdaLomo(cfg, ADA_SHAPES)
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in ADA_SHAPES])])
    for t in range(1, ADA_STEPS + 1):
        # the collective sums the ranks' fp32 gradients in fp32 (<= 1 rounding, far
        # inside the tolerance); the oracle sums them in fp64
        g = sum(_ada_grads(k, t).astype(np.float64) for k in range(world))
        scale = 1.0 if clip is None else O.orc.orc_clip_scale(
            O.orc.orc_sumsq_f64(O._ptr(g), g.size), clip)
        for k in range(len(ADA_SHAPES)):
            gk = np.ascontiguousarray(g[offs[k]:offs[k + 1]] * scale)
            r.apply(k, ps[k], gk, ADA_LR)
    want = np.concatenate(ps)
    rms = float(np.sqrt(np.mean(np.concatenate(p0) ** 2)))
    for rank in range(world):
        got = res[rank].astype(np.float64)
        err = np.abs(got - want) / np.maximum(np.abs(want), rms)
        assert err.max() <= 1e-5, (rank, err.max())
    for rank in range(1, world):  # every replica identical
        assert np.array_equal(res[0], res[rank])


@needs_ref
@pytest.mark.parametrize("world", [2, 3])
def test_zero_sharded_lomo_clip_processes_match_reference(world):
    check_zero_sharded_lomo(world, "gloo")


def check_zero_sharded_lomo(world, backend):
    clip = 0.05
    res = _run("lomo32", world, clip, backend)
    want = O.synth(LOMO_P, 61, 0, 0, 0, 0, -6, 0, False).astype(np.float64)
    p0 = want.copy()
    for t in range(1, LOMO_STEPS + 1):
        g = sum(_lomo_grad(k, t) for k in range(world)).astype(np.float64)
        O.ref_lomo_fused([want], [g], LOMO_LR, clip)
    rms = float(np.sqrt(np.mean(p0 ** 2)))
    for rank in range(world):
        err = np.abs(res[rank].astype(np.float64) - want) / np.maximum(np.abs(want), rms)
        assert err.max() <= 1e-5, (rank, err.max())
    for rank in range(1, world):
        assert np.array_equal(res[0], res[rank])


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lomo_bf16_clip_processes_match_restatement(world):
    """C5: bf16 owned shards (fp32 arithmetic, RNE store), the global norm from one fp64
    all-reduce of the ranks' partial sums; vs the bf16 restatement with the serial
    clip scale -- equal up to one bf16 ulp where the two fp64 norms (different
    summation order) round the fp32 factor differently."""
    check_sharded_lomo_bf16(world, "gloo")


def check_sharded_lomo_bf16(world, backend):
    clip = 0.05
    res = _run("lomo_bf16", world, clip, backend)
    from paper_2312_00407_b200 import zero

    want = O.f32_to_bf16(O.synth(LOMO_P, 62, 0, 0, 0, 0, -6, 0, False))
    for t in range(1, LOMO_STEPS + 1):
        gb = O.f32_to_bf16(O.synth(LOMO_P, 62, 1, 0, t, 0, -7, 10, False))
        g64 = O.bf16_to_f32(gb).astype(np.float64)
        scale = O.orc.orc_clip_scale(O.orc.orc_sumsq_f64(O._ptr(g64), g64.size), clip)
        O.orc.orc_lomo_bf16(O._ptr(want), O._ptr(gb), LOMO_P, LOMO_LR, scale)
    plan = zero.ZeroPlan.make(LOMO_P, world)
    got = np.concatenate([res[r] for r in range(world)])
    assert got.size == LOMO_P and plan.offsets[-1] == LOMO_P
    d = np.abs(got.astype(np.int32) - want.astype(np.int32))
    assert d.max() <= 1 and np.mean(d == 0) >= 0.999, (d.max(), np.mean(d == 0))
