"""Multi-rank host logic of the ZeRO sharder on CPU (gloo, world size 2 and 3):
ZeroPlan bookkeeping, reduce-scatter / all-gather of owned slices, and the sharded
step == the serial FlatOptimizer step on the summed gradient (SerialBaseline,
tests/serial_ref.hpp:34-70).  The per-shard update is the oracle here (no GPU);
on the GPU it is the CUDA FlatOptimizer (tests/test_gpu_zero.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 4
CASES = {2: [(1000, 0), (1001, 2)], 3: [(10, 3), (1000, 1)]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _grad(P, rank, t, dtype=np.float64):
    import oracle as O

    return O.synth(P, 3, 1, rank, t, 0, -7, 0, False, dtype)


def _worker(rank, world, port, out_q):
    import sys

    for p in (ROOT, os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    import oracle as O
    from paper_2312_00407_b200 import zero
    from paper_2312_00407_b200.optim import OptimizerConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        for P, kind in CASES[world]:
            cfg = OptimizerConfig.defaults_for(kind)
            cfg.weight_decay = 0.01
            plan = zero.ZeroPlan.make(P, world, 2)
            lo, hi = plan.owned_range(rank)
            orc = O.OracleFlat(cfg, hi - lo, np.float64)

            def local(p_owned, g_owned, lr, p_out, orc=orc):
                a = p_owned.numpy()
                orc.step(a, np.ascontiguousarray(g_owned.numpy()), lr)

            params = torch.from_numpy(O.synth(P, 3, 0, 0, 0, 0, -6, 0, False, np.float64))
            opt = zero.ZeroShardedOptimizer(cfg, P, local_step=local)
            assert opt.owned_range() == (lo, hi)
            for t in range(1, STEPS + 1):
                opt.step(params, torch.from_numpy(_grad(P, rank, t)), 1e-3)
            out[(P, kind)] = (params.numpy().copy(), (lo, hi), dict(orc.state))

        # the other ZeRO stages of parallel.cpp:637-672 on the first case
        P, kind = CASES[world][0]
        for stage in (0, 1, 3):
            cfg = OptimizerConfig.defaults_for(kind)
            cfg.weight_decay = 0.01
            plan = zero.ZeroPlan.make(P, world, stage)
            lo, hi = plan.owned_range(rank) if stage >= 1 else (0, P)
            orc = O.OracleFlat(cfg, hi - lo, np.float64)

            def local_s(p_owned, g_owned, lr, p_out, orc=orc):
                orc.step(p_owned.numpy(), np.ascontiguousarray(g_owned.numpy()), lr)

            full = torch.from_numpy(O.synth(P, 3, 0, 0, 0, 0, -6, 0, False, np.float64))
            params = full[lo:hi].clone() if stage == 3 else full
            opt = zero.ZeroShardedOptimizer(cfg, P, stage=stage, local_step=local_s)
            assert opt.owned_range() == (lo, hi)
            for t in range(1, STEPS + 1):
                opt.step(params, torch.from_numpy(_grad(P, rank, t)), 1e-3)
            out[("stage", stage)] = (params.numpy().copy(), (lo, hi))

        if world == 2:
            # mixed precision: bf16 replicated params, fp32 master + state per shard
            P = 1000
            cfg = OptimizerConfig.defaults_for(0)
            orc = O.OracleFlat(cfg, 500, np.float32)

            def local32(master, g_owned, lr, p_out):
                a = master.numpy()
                orc.step(a, np.ascontiguousarray(g_owned.numpy()), lr)
                p_out.copy_(master.to(torch.bfloat16))

            p0 = torch.from_numpy(O.synth(P, 3, 0, 0, 0, 0, -6, 0, False, np.float32))
            params = p0.to(torch.bfloat16)
            opt = zero.ZeroShardedOptimizer(cfg, P, local_step=local32, mixed=True,
                                            master_init=p0)
            for t in range(1, STEPS + 1):
                g = torch.from_numpy(_grad(P, rank, t, np.float32))
                opt.step(params, g, 1e-3)
            out["mixed"] = params.float().numpy().copy()

            # LOMO with the global grad-norm clip across shards
            ops = type("Ops", (), {})
            ops.sumsq = staticmethod(lambda g, stream=None: torch.tensor(
                float(np.dot(g.numpy(), g.numpy())), dtype=torch.float64))
            ops.apply = staticmethod(lambda p, g, lr, sc, st=None: p.sub_(lr * sc * g))

            def apply_clipped(p, g, lr, s, clip, st=None):
                p.sub_((lr * O.orc.orc_clip_scale(float(s.item()), clip)) * g)

            ops.apply_clipped = staticmethod(apply_clipped)
            lo, hi = zero.ZeroPlan.make(1001, 2).owned_range(rank)
            pf = O.synth(1001, 3, 0, 9, 0, 0, -6, 0, False, np.float64)
            gf = O.synth(1001, 3, 1, 9, 1, 0, -2, 0, False, np.float64)
            lp = torch.from_numpy(pf[lo:hi].copy())
            s = zero.sharded_lomo_step(lp, torch.from_numpy(gf[lo:hi].copy()), 0.1, 0.5, ops=ops)
            out["lomo"] = (lp.numpy().copy(), float(s.item()), (lo, hi))
        out_q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _serial(P, world, kind, dtype=np.float64, wd=0.01):
    import oracle as O
    from paper_2312_00407_b200.optim import OptimizerConfig

    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = wd
    p = O.synth(P, 3, 0, 0, 0, 0, -6, 0, False, dtype)
    o = O.OracleFlat(cfg, P, dtype)
    for t in range(1, STEPS + 1):
        g = _grad(P, 0, t, dtype)
        for r in range(1, world):
            g = g + _grad(P, r, t, dtype)
        o.step(p, g.astype(dtype), 1e-3)
    return p, o.state


@pytest.fixture(scope="module")
def world2():
    return _run(2)


@pytest.fixture(scope="module")
def world3():
    return _run(3)


def _check(res, world):
    for (P, kind) in CASES[world]:
        want_p, want_state = _serial(P, world, kind)
        ranges = []
        for rank in range(world):
            params, (lo, hi), state = res[rank][(P, kind)]
            ranges.append((lo, hi))
            if world == 2:
                assert np.array_equal(params, want_p)  # a + b is exact-commutative
            else:
                np.testing.assert_allclose(params, want_p, rtol=1e-13, atol=1e-18)
            for name, buf in state.items():  # state only for the owned slice
                np.testing.assert_allclose(buf, want_state[name][lo:hi], rtol=1e-12,
                                           atol=1e-300)
        assert ranges[0][0] == 0 and ranges[-1][1] == P
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
        if (world, P) == (3, 10):
            assert [b - a for a, b in ranges] == [4, 3, 3]  # ZeroPlan, trailing smaller


def _check_stages(res, world):
    P, kind = CASES[world][0]
    want, _ = _serial(P, world, kind)
    for rank in range(world):
        for stage in (0, 1, 3):
            got, (lo, hi) = res[rank][("stage", stage)]
            ref = want[lo:hi] if stage == 3 else want
            if world == 2:
                assert np.array_equal(got, ref), stage
            else:
                np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-18)


def test_zero_stages_0_1_3_equal_serial(world2, world3):
    """parallel.cpp:637-672: AR + full step (0), AR + owned step + AG (1), RS + owned
    step on the stage-3 shard (3) -- the same trajectory as stage 2 and serial."""
    _check_stages(world2, 2)
    _check_stages(world3, 3)


def test_sharded_step_equals_serial_world2(world2):
    _check(world2, 2)


def test_sharded_step_equals_serial_world3_uneven(world3):
    _check(world3, 3)


def test_mixed_master_bf16_replicas(world2):
    import oracle as O

    want, _ = _serial(1000, 2, 0, np.float32, wd=0.0)
    for rank in range(2):
        got = world2[rank]["mixed"]
        assert np.array_equal(got.astype(np.float32).view(np.uint32) >> 16,
                              O.f32_to_bf16(want).astype(np.uint32))


def test_sharded_lomo_clip_uses_global_norm(world2):
    import oracle as O

    g = O.synth(1001, 3, 1, 9, 1, 0, -2, 0, False, np.float64)
    pf = O.synth(1001, 3, 0, 9, 0, 0, -6, 0, False, np.float64)
    total = float(np.dot(g, g))
    scale = O.orc.orc_clip_scale(total, 0.5)
    for rank in range(2):
        lp, s, (lo, hi) = world2[rank]["lomo"]
        assert s == pytest.approx(total, rel=1e-13)  # every rank sees the global sum
        np.testing.assert_allclose(lp, pf[lo:hi] - (0.1 * scale) * g[lo:hi], rtol=1e-13)


def _mismatch_worker(rank, world, port, out_q):
    import sys

    for p in (ROOT, os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    from paper_2312_00407_b200 import optim, zero
    from paper_2312_00407_b200.optim import OptimizerConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = OptimizerConfig.defaults_for(0)
        try:  # rank 1 was handed a different flat length: every rank must fail fast
            zero.ZeroShardedOptimizer(cfg, 1000 + rank, local_step=lambda *a: None)
            out_q.put((rank, "no error"))
        except optim.ProtocolError as e:
            out_q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_plan_mismatch_fails_fast_on_every_rank():
    """comm.cpp:160-167 length-mismatch abort + comm.cpp:337-360 rank attribution."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mismatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert res[r].startswith(f"[rank {r}] ZeroShardedOptimizer: ranks [1] disagree"), res[r]
        assert "1000" in res[r] and "1001" in res[r]
