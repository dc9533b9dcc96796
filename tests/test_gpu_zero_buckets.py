"""The bucketed, double-buffered stage-2 step (mco_zb_*, zero.BucketedZeroOptimizer;
SURVEY 8(e) C4) and the NCCL failure handling (mco_comm_create_timeout / abort).

One GPU: the collectives run over a world-1 NCCL communicator (identities), so these
pin the bucket / piece / state-offset bookkeeping, the once-per-step ++t, the
double-buffered staging slots, the mixed (bf16 replica + fp32 master) and ring modes:
every form is bit-identical to the plain FlatOptimizer step.  The multi-rank piece
layout is pinned against ZeroPlan in tests/test_zero_buckets_plan.py (CPU); the C4
per-rank footprints at N = 2 / 8 are allocated and stepped in test_gpu_00_footprint.py."""
import pytest

import oracle as O
from paper_2312_00407_b200 import optim, zero
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

P = 100003


def cfg_for(kind):
    c = OptimizerConfig.defaults_for(kind)
    c.weight_decay = 0.01
    return c


def grads(t, n=P):
    return torch.from_numpy(O.synth(n, 9, 1, 0, t, 0, -7, 10, False)).cuda()


def bits(t):
    return t.view(torch.int32) if t.dtype == torch.float32 else t.view(torch.int16)


@pytest.fixture(scope="module")
def comm():
    return zero.NcclComm()


@pytest.mark.parametrize("kind", [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA])
@pytest.mark.parametrize("bucket", [0, 4096, 33331])
def test_bucketed_f32_equals_flat_step(comm, kind, bucket):
    cfg = cfg_for(kind)
    zb = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=bucket)
    ref = optim.FlatOptimizer(cfg, P)
    p = torch.from_numpy(O.synth(P, 9, 0, 0, 0, 0, -6, 0, False)).cuda()
    q = p.clone()
    for t in range(1, 13):  # past Sophia's refresh at t = 11
        g = grads(t)
        zb.step(p, g, 1e-3)
        ref.step(q, g, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(bits(p), bits(q))
    assert zb.steps_taken() == 12
    if bucket:
        assert zb.nbuckets == -(-P // zb.bucket_elems) and zb.bucket_elems % 8 == 0
    for (na, a), (nb, b) in zip(zb.buffers(), ref.buffers()):
        assert na == nb and torch.equal(bits(a), bits(b)), na


@pytest.mark.parametrize("kind", [Kind.ADAN, Kind.SOPHIA])
def test_bucketed_mixed_equals_step_mixed(comm, kind):
    """C4 layout: fp32 master of the owned pieces, bf16 replicas written by the update
    and all-gathered; bf16 gradients."""
    cfg = cfg_for(kind)
    zb = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=8192,
                                    grad_dtype=torch.bfloat16, replica_dtype=torch.bfloat16)
    ref = optim.FlatOptimizer(cfg, P)
    p0 = torch.from_numpy(O.synth(P, 9, 0, 0, 0, 0, -6, 0, False)).cuda()
    zb.load_master(p0)
    master = p0.clone()
    rep = torch.zeros(P, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros_like(rep)
    for t in range(1, 4):
        g = grads(t).to(torch.bfloat16)
        zb.step(rep, g, 1e-3)
        ref.step_mixed(master, g, out, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(bits(rep), bits(out))
    assert torch.equal(bits(zb.master()), bits(master))


def test_bucketed_streaming_staging_slots_equal_whole_step(comm):
    """Gradients produced bucket by bucket into the library's double-buffered staging
    slots (no full-length gradient handed in) == the whole-buffer step."""
    cfg = cfg_for(Kind.ADAMW)
    a = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=10000)
    b = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=10000)
    pa = torch.from_numpy(O.synth(P, 9, 0, 0, 0, 0, -6, 0, False)).cuda()
    pb = pa.clone()
    B = a.bucket_elems
    for t in range(1, 4):
        g = grads(t)
        a.step(pa, g, 1e-3)
        b.begin(pb, 1e-3)
        for k in reversed(range(b.nbuckets)):
            buf = b.grad_buffer(k)
            buf.copy_(g[k * B:k * B + buf.numel()])
            b.grad_ready(k)
        b.end()
    torch.cuda.synchronize()
    assert torch.equal(bits(pa), bits(pb))


def test_bucketed_ring_mode_gathers_each_bucket(comm):
    """Ring mode (stage-3 layout): no replica buffer; bucket k's gathered bf16
    parameters == the bf16 parameters of the plain mixed step."""
    cfg = cfg_for(Kind.SOPHIA)
    zb = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=16384,
                                    replica_dtype=torch.bfloat16)
    ref = optim.FlatOptimizer(cfg, P)
    p0 = torch.from_numpy(O.synth(P, 9, 0, 0, 0, 0, -6, 0, False)).cuda()
    zb.load_master(p0)
    master, out = p0.clone(), torch.zeros(P, dtype=torch.bfloat16, device="cuda")
    B = zb.bucket_elems
    for t in range(1, 3):
        g = grads(t)
        ref.step_mixed(master, g, out, 1e-3)
        zb.begin(None, 1e-3)
        got = {}
        for k in range(zb.nbuckets):  # consume bucket k-1 while k is reduced (forward)
            zb.grad_ready(k, g[k * B:])
            if k >= 1:
                got[k - 1] = zb.gathered(k - 1).clone()
        zb.end()
        got[zb.nbuckets - 1] = zb.gathered(zb.nbuckets - 1).clone()
        torch.cuda.synchronize()
        for k, v in got.items():
            assert torch.equal(bits(v), bits(out[k * B:k * B + v.numel()])), (t, k)


def test_bucketed_rejects_bad_use(comm):
    cfg = cfg_for(Kind.ADAMW)
    zb = zero.BucketedZeroOptimizer(cfg, 1000, comm, bucket_elems=256)
    p = torch.zeros(1000, device="cuda")
    with pytest.raises(optim.ContractError, match="mco_zb_begin first"):
        zb.grad_ready(0, torch.zeros(1000, device="cuda"))
    zb.begin(p, 1e-3)
    zb.grad_ready(1, torch.zeros(1000, device="cuda"))
    with pytest.raises(optim.ContractError, match="already reduced"):
        zb.grad_ready(1, torch.zeros(1000, device="cuda"))
    with pytest.raises(optim.ContractError, match="buckets reduced"):
        zb.end()
    with pytest.raises(optim.ContractError, match="ring mode"):
        zb.begin(None, 1e-3)  # f32 replicas: the parameters ARE the replicas
    with pytest.raises(optim.ContractError, match="fused"):
        zero.BucketedZeroOptimizer(OptimizerConfig.defaults_for(Kind.LOMO), 1000, comm)


@pytest.mark.timeout(300)
def test_nccl_missing_rank_times_out_and_aborts():
    """comm.cpp:126-132 / 330-348: a communicator of 2 ranks whose rank 1 never joins
    -- init gives up at the deadline, aborts, and names this rank (no hang)."""
    import time

    t0 = time.time()
    with pytest.raises(optim.ProtocolError, match=r"\[rank 0 of 2\].*(join|timed out)"):
        zero.NcclComm(world=2, rank=0, timeout_s=5.0)
    assert time.time() - t0 < 120


