"""Bucketed, backward-overlapped ZeRO step (overlap.OverlappedZeroOptimizer, SURVEY
8(f) f4) on one B200: the sm_100a FlatOptimizer runs per bucket on a side stream
while backward continues; the result is bit-identical to one FlatOptimizer step over
the whole flat gradient (the update is elementwise, pieces are sub-ranges)."""
import pytest

from paper_2312_00407_b200 import optim, overlap
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def deep_mlp(seed, width=1024, depth=8):
    g = torch.Generator().manual_seed(seed)
    layers = []
    for _ in range(depth):
        layers += [torch.nn.Linear(width, width), torch.nn.GELU()]
    m = torch.nn.Sequential(*layers)
    with torch.no_grad():
        for p in m.parameters():
            p.copy_(torch.randn(p.shape, generator=g) * 0.03)
    return m.cuda()


def batch(t, width=1024):
    g = torch.Generator().manual_seed(500 + t)
    return torch.randn(256, width, generator=g).cuda(), torch.randn(256, width, generator=g).cuda()


@pytest.mark.parametrize("kind", [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA])
def test_overlapped_equals_flat_step(kind):
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 0.01
    a, b = deep_mlp(3), deep_mlp(3)
    ov = overlap.OverlappedZeroOptimizer(cfg, list(a.parameters()), bucket_elems=1 << 20)
    assert len(ov.buckets) > 4
    pb = list(b.parameters())
    ref = optim.FlatOptimizer(cfg, sum(p.numel() for p in pb))
    flat_b = torch.cat([p.detach().reshape(-1) for p in pb])
    for t in range(1, 5):
        x, y = batch(t)
        ov.backward_step(lambda: ((a(x) - y) ** 2).mean(), 1e-3)
        assert ov.launched_in_backward == len(ov.buckets)
        # reference: plain backward, flatten, one flat step, scatter back
        with torch.no_grad():
            off = 0
            for p in pb:
                p.copy_(flat_b[off:off + p.numel()].view_as(p))
                off += p.numel()
        b.zero_grad()
        ((b(x) - y) ** 2).mean().backward()
        g = torch.cat([p.grad.reshape(-1) for p in pb])
        ref.step(flat_b, g, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(ov.flat_params, flat_b)
    st = ov.extract_state()
    assert st["steps"] == 4
    for name, buf in ref.buffers():
        assert torch.equal(st["buffers"][name], buf), name


def test_updates_overlap_backward():
    """The first buckets' updates complete on the side stream before backward ends."""
    cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
    m = deep_mlp(5, width=2048, depth=12)
    ov = overlap.OverlappedZeroOptimizer(cfg, list(m.parameters()), bucket_elems=1 << 22)
    x, y = batch(1, 2048)
    for _ in range(2):  # warm-up (allocator, kernels)
        ov.backward_step(lambda: ((m(x) - y) ** 2).mean(), 1e-4)
    torch.cuda.synchronize()
    ov.begin(1e-4)
    loss = ((m(x) - y) ** 2).mean()
    loss.backward()
    end = torch.cuda.Event(enable_timing=True)
    end.record()  # compute stream: backward done
    ov.finish()
    torch.cuda.synchronize()
    assert ov.launched_in_backward == len(ov.buckets)
    first = ov.bucket_events[0]
    assert first.elapsed_time(end) > 0.0  # bucket 0 finished before backward did


def test_state_round_trip_and_grad_rebinding():
    cfg = OptimizerConfig.defaults_for(Kind.ADAN)
    m = deep_mlp(9, width=256, depth=3)
    ov = overlap.OverlappedZeroOptimizer(cfg, list(m.parameters()), bucket_elems=70000)
    x, y = batch(2, 256)
    ov.backward_step(lambda: ((m(x) - y) ** 2).mean(), 1e-3)
    st = ov.extract_state()
    m2 = deep_mlp(9, width=256, depth=3)
    ov2 = overlap.OverlappedZeroOptimizer(cfg, list(m2.parameters()), bucket_elems=1 << 30)
    ov2.load_state(st)  # different bucketing, same owned slice
    with torch.no_grad():
        ov2.flat_params.copy_(ov.flat_params)
    for p in m.parameters():
        p.grad = None  # a user dropping grads: begin() rebinds the flat views
    for o, mm in ((ov, m), (ov2, m2)):
        o.backward_step(lambda: ((mm(x) - y) ** 2).mean(), 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(ov.flat_params, ov2.flat_params)
