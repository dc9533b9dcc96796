"""GPU tests of the ZeRO sharder.  Only one GPU is available, so the multi-rank
peer-memory kernel is exercised with N *virtual* ranks on one device: N separate
flat grad buffers and N parameter replicas, the kernel launched once per rank
with that rank's ZeroPlan range -- the same pointers-to-every-rank layout the
IPC-mapped multi-GPU run uses.  The NCCL paths run at world size 1."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200 import optim, zero
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cfg_for(kind):
    c = OptimizerConfig.defaults_for(kind)
    c.weight_decay = 0.01
    return c


@pytest.mark.parametrize("kind", [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA])
@pytest.mark.parametrize("world,P", [(2, 1 << 16), (4, 100003), (8, 999)])
def test_peer_kernel_virtual_ranks_equals_serial(kind, world, P):
    cfg = cfg_for(kind)
    plan = zero.ZeroPlan.make(P, world)
    p0 = O.synth(P, 5, 0, 0, 0, 0, -6, 0, False)
    replicas = [dev(p0) for _ in range(world)]
    opts = [optim.FlatOptimizer(cfg, plan.part_sizes[r]) for r in range(world)]
    serial, ps = O.OracleFlat(cfg, P, np.float32), p0.copy()
    for t in range(1, 4):
        gs = [O.synth(P, 5, 1, r, t, 0, -7, 10, False) for r in range(world)]
        grads = [dev(g) for g in gs]
        for r in range(world):  # rank r's kernel, master = its own f32 replica slice
            lo, hi = plan.owned_range(r)
            opts[r].step_peers(grads, replicas, replicas[r][lo:hi], lo, hi - lo, 1e-3)
        gsum = gs[0].copy()
        for g in gs[1:]:
            gsum = gsum + g  # the kernel's rank-order fp32 sum
        serial.step(ps, gsum, 1e-3)
    torch.cuda.synchronize()
    for r in range(world):  # every replica holds the full, bit-identical result
        assert np.array_equal(replicas[r].cpu().numpy().view(np.uint32), ps.view(np.uint32))
    for r in range(world):
        lo, hi = plan.owned_range(r)
        for name, buf in opts[r].buffers():
            assert np.array_equal(buf.cpu().numpy().view(np.uint32),
                                  serial.state[name][lo:hi].view(np.uint32)), (r, name)


def test_peer_kernel_bf16_replicas_and_grads():
    world, P = 4, 50000
    cfg = cfg_for(Kind.ADAN)
    plan = zero.ZeroPlan.make(P, world)
    p0 = O.synth(P, 6, 0, 0, 0, 0, -6, 0, False)
    replicas = [dev(O.f32_to_bf16(p0)).view(torch.bfloat16) for _ in range(world)]
    masters = [dev(p0[plan.offsets[r]:plan.offsets[r + 1]]) for r in range(world)]
    opts = [optim.FlatOptimizer(cfg, plan.part_sizes[r]) for r in range(world)]
    serial, ps = O.OracleFlat(cfg, P, np.float32), p0.copy()
    for t in (1, 2):
        gb = [O.synth(P, 6, 1, r, t, 0, -7, 10, False, "bf16") for r in range(world)]
        grads = [dev(g).view(torch.bfloat16) for g in gb]
        for r in range(world):
            lo, hi = plan.owned_range(r)
            opts[r].step_peers(grads, replicas, masters[r], lo, hi - lo, 1e-3)
        gsum = O.bf16_to_f32(gb[0]).copy()
        for g in gb[1:]:
            gsum = gsum + O.bf16_to_f32(g)
        serial.step(ps, gsum, 1e-3)
    torch.cuda.synchronize()
    want = O.f32_to_bf16(ps)
    for r in range(world):
        assert np.array_equal(replicas[r].view(torch.int16).cpu().numpy().view(np.uint16), want)
    got_master = np.concatenate([m.cpu().numpy() for m in masters])
    assert np.array_equal(got_master.view(np.uint32), ps.view(np.uint32))


@pytest.fixture(scope="module")
def nccl1():
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_zero_sharded_nccl_world1_equals_flat(nccl1):
    P = 123457
    cfg = cfg_for(Kind.ADAMW)
    p0 = O.synth(P, 7, 0, 0, 0, 0, -6, 0, False)
    a, b = dev(p0), dev(p0)
    z = zero.ZeroShardedOptimizer(cfg, P)
    f = optim.FlatOptimizer(cfg, P)
    for t in (1, 2):
        g = dev(O.synth(P, 7, 1, 0, t, 0, -7, 10, False))
        z.step(a, g, 1e-3)
        f.step(b, g, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    st = z.extract_state()
    z2 = zero.ZeroShardedOptimizer(cfg, P)
    z2.load_state(st)
    assert z2.opt.steps_taken() == 2
    assert all(torch.equal(x, y) for (_, x), (_, y) in zip(z.opt.buffers(), z2.opt.buffers()))


def test_peer_sharded_optimizer_world1(nccl1):
    P = 77777
    cfg = cfg_for(Kind.SOPHIA)
    ps = zero.PeerShardedOptimizer(cfg, P)
    p0 = O.synth(P, 8, 0, 0, 0, 0, -6, 0, False)
    ps.params.copy_(dev(p0))
    serial, want = O.OracleFlat(cfg, P, np.float32), p0.copy()
    for t in (1, 2, 3):
        g = O.synth(P, 8, 1, 0, t, 0, -7, 10, False)
        ps.grads.copy_(dev(g))
        ps.step(1e-3)
        serial.step(want, g, 1e-3)
    torch.cuda.synchronize()
    assert np.array_equal(ps.params.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_sharded_lomo_clip_world1(nccl1):
    P = 65536
    p0 = O.synth(P, 9, 0, 0, 0, 0, -6, 0, False, "bf16")
    g = O.synth(P, 9, 1, 0, 1, 0, -7, 10, False, "bf16")
    tp = dev(p0).view(torch.bfloat16)
    s = zero.sharded_lomo_step(tp, dev(g).view(torch.bfloat16), 1e-2, 0.01)
    total = O.orc.orc_sumsq_bf16(O._ptr(g), P)
    assert s.item() == pytest.approx(total, rel=1e-10)
    scale = O.orc.orc_clip_scale(total, 0.01)
    want = p0.copy()
    O.orc.orc_lomo_bf16(O._ptr(want), O._ptr(g), P, 1e-2, scale)
    torch.cuda.synchronize()
    got = tp.view(torch.int16).cpu().numpy().view(np.uint16)
    # the device norm differs from the sequential one in the last bits -> scale
    # may differ by 1 ulp; bf16 results may then differ by 1 ulp in rare ties
    assert np.mean(got != want) < 1e-3


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("world", [2, 3, 4])
def test_row_sharded_adalomo_virtual_ranks_equals_serial(world):
    """Row-split AdaLomo (column-statistic and sum-u^2 all-reduces) == serial AdaLomo
    (the compiled reference) on the whole matrices."""
    from test_gpu_fused import SHAPES, ada_inputs, ada_tol_ok

    shapes = SHAPES + [(7, 24), (2, 16)]  # rows < world on some ranks
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ranks = [zero.RowShardedAdaLomo(cfg, shapes, rank=r, world=world) for r in range(world)]
    ps, gs = ada_inputs(shapes, 3)
    p0 = [x.copy() for x in ps]
    flat_p = dev(np.concatenate(ps).astype(np.float32))
    ref = O.RefAdaLomo(cfg, shapes)
    for t in range(3):
        flat_g = dev(np.concatenate(gs[t]).astype(np.float32))
        lp = [rk.scatter(flat_p) for rk in ranks]
        lg = [rk.scatter(flat_g) for rk in ranks]
        for phase in (1, 2, 3):
            for r, rk in enumerate(ranks):
                rk.state.phase(phase, lp[r], lg[r], 5e-3)
            if phase < 3:  # the all-reduce, in rank order
                pays = [rk.state.payload(phase - 1) for rk in ranks]
                total = pays[0].clone()
                for x in pays[1:]:
                    total += x
                for x in pays:
                    x.copy_(total)
        for r, rk in enumerate(ranks):
            rk.gather_into(lp[r], flat_p)
        for k in range(len(shapes)):
            ref.apply(k, ps[k], gs[t][k], 5e-3)
    torch.cuda.synchronize()
    got = flat_p.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
    for k in range(len(shapes)):
        ok, e = ada_tol_ok(got[offs[k]:offs[k + 1]], ps[k], p0[k])
        assert ok, (k, shapes[k], e)


def test_row_sharded_adalomo_world1_nccl(nccl1):
    from test_gpu_fused import SHAPES, ada_inputs

    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    rs = zero.RowShardedAdaLomo(cfg, SHAPES)
    plain = optim.AdaLomoState(cfg, SHAPES)
    ps, gs = ada_inputs(SHAPES, 2)
    a = dev(np.concatenate(ps).astype(np.float32))
    b = a.clone()
    for t in range(2):
        g = dev(np.concatenate(gs[t]).astype(np.float32))
        rs.step(a, g, 1e-2)
        plain.apply_all(b, g, 1e-2)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def _ipc_worker(rank, world, port, kind, P, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "oracle")):
        sys.path.insert(0, p)
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2312_00407_b200 import zero
    from paper_2312_00407_b200.optim import OptimizerConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        cfg = OptimizerConfig.defaults_for(kind)
        cfg.weight_decay = 0.0
        if kind == 4:
            cfg.clip_threshold = 0.05
        ps = zero.PeerShardedOptimizer(cfg, P)
        ps.params.copy_(torch.from_numpy(O.synth(P, 21, 0, 0, 0, 0, -6, 0, False)).cuda())
        for t in (1, 2, 3):
            g = O.synth(P, 21, 1, rank, t, 0, -7, 10, False)
            ps.grads.copy_(torch.from_numpy(g).cuda())
            torch.cuda.synchronize()
            ps.step(1e-3)
        torch.cuda.synchronize()
        q.put((rank, ps.params.cpu().numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", [Kind.ADAMW, Kind.LOMO])
def test_peer_sharded_two_processes_ipc_one_gpu(kind):
    """Two OS processes on one B200, each mapping the other's buffers through CUDA
    IPC: the real multi-process PeerShardedOptimizer path (gloo control plane)."""
    import torch.multiprocessing as mp

    P, world = 100001, 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, int(kind), P, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = O.synth(P, 21, 0, 0, 0, 0, -6, 0, False)
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 0.0
    orc = O.OracleFlat(cfg, P, np.float32) if kind != Kind.LOMO else None
    for t in (1, 2, 3):
        g = O.synth(P, 21, 1, 0, t, 0, -7, 10, False) + O.synth(P, 21, 1, 1, t, 0, -7, 10, False)
        if orc is not None:
            orc.step(want, g, 1e-3)
        else:
            scale = O.orc.orc_clip_scale(float(np.dot(g.astype(np.float64), g)), 0.05)
            O.orc.orc_lomo_f32(O._ptr(want), O._ptr(g), P, 1e-3, scale)
    for r in range(world):
        if orc is not None:
            assert np.array_equal(res[r].view(np.uint32), want.view(np.uint32))
        else:  # the clip norm is summed in a different order than the oracle's
            np.testing.assert_allclose(res[r], want, rtol=0, atol=1e-7)
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("algo", ["even", "p2p"])
@pytest.mark.parametrize("kind", [Kind.ADAMW, Kind.ADAN])
def test_native_nccl_shard_step_world1(monkeypatch, algo, kind):
    """mco_shard_step through the library's own NCCL communicator (one rank: the
    collectives are identities) == the plain FlatOptimizer step, bit for bit, on both
    the reduce-scatter / all-gather path and the per-part reduce / broadcast path."""
    if algo == "p2p":
        monkeypatch.setenv("MCO_SHARD_ALGO", "p2p")
    n = 100003
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 0.01
    comm = zero.NcclComm()
    nz = zero.NativeZeroOptimizer(cfg, n, comm)
    ref = optim.FlatOptimizer(cfg, n)
    p0 = O.synth(n, 5, 0, 0, 0, 0, -6, 0, False)
    a, b = torch.from_numpy(p0.copy()).cuda(), torch.from_numpy(p0.copy()).cuda()
    for t in (1, 2, 3):
        g = torch.from_numpy(O.synth(n, 5, 1, 0, t, 0, -7, 10, False)).cuda()
        g_keep = g.clone()
        nz.step(a, g, 1e-3)
        ref.step(b, g_keep, 1e-3)
        torch.cuda.synchronize()
        assert torch.equal(g, g_keep)  # const gradients: reduced into the comm's scratch
    assert torch.equal(a, b)
    for (n1, x), (n2, y) in zip(nz.opt.buffers(), ref.buffers()):
        assert n1 == n2 and torch.equal(x, y)
    comm.check()
    t = torch.arange(10, dtype=torch.float64, device="cuda")
    comm.allreduce_sum(t)
    torch.cuda.synchronize()
    assert torch.equal(t, torch.arange(10, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("algo", ["rs_ag", "p2p"])
@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16], ids=["f32g", "bf16g"])
def test_native_nccl_shard_step_mixed_world1(monkeypatch, algo, gdt):
    """mco_shard_step_mixed (fp32 master + state, bf16 replicas, bf16 all-gather) with
    one rank == FlatOptimizer.step_mixed on the whole vector, master and replicas bit for
    bit; the master follows the replica slice's alignment phase."""
    if algo == "p2p":
        monkeypatch.setenv("MCO_SHARD_ALGO", "p2p")
    n = 100003
    cfg = OptimizerConfig.defaults_for(Kind.ADAN)
    cfg.weight_decay = 0.01
    p0 = torch.from_numpy(O.synth(n, 9, 0, 0, 0, 0, -6, 0, False)).cuda()
    comm = zero.NcclComm()
    nz = zero.NativeZeroOptimizer(cfg, n, comm, mixed=True, master_init=p0)
    ref = optim.FlatOptimizer(cfg, n)
    rep_buf = torch.empty(n + 3, dtype=torch.bfloat16, device="cuda")
    rep = rep_buf[3:]  # replicas at an odd phase: the master must follow it
    rep.copy_(p0.bfloat16())
    master = p0.clone()
    rep_ref = rep.clone()
    for t in (1, 2, 3):
        g = torch.from_numpy(O.synth(n, 9, 1, 0, t, 0, -7, 10, False)).cuda().to(gdt)
        nz.step(rep, g, 1e-3)
        ref.step_mixed(master, g, rep_ref, 1e-3)
    torch.cuda.synchronize()
    assert zero.elem_phase(nz.master) == zero.elem_phase(rep)
    assert torch.equal(nz.master, master)
    assert torch.equal(rep, rep_ref)
    comm.check()


def test_native_shard_step_contract_errors():
    comm = zero.NcclComm()
    nz = zero.NativeZeroOptimizer(OptimizerConfig.defaults_for(Kind.ADAMW), 1000, comm)
    with pytest.raises(optim.ContractError):
        nz.step(torch.zeros(999, device="cuda"), torch.zeros(999, device="cuda"), 1e-3)
    from paper_2312_00407_b200 import _lib
    import ctypes as C

    bad = optim.FlatOptimizer(OptimizerConfig.defaults_for(Kind.ADAMW), 10)
    p = torch.zeros(1000, device="cuda")
    st = _lib.lib.mco_shard_step(bad._h, comm._h, p.data_ptr(), 0, p.data_ptr(), 0, 1000,
                                 C.c_double(1e-3), None)
    assert st == _lib.MCO_CONTRACT
    assert "ZeroPlan gives rank 0 1000" in _lib.lib.mco_last_error().decode()
