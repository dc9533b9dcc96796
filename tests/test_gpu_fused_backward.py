"""Backward-fused LOMO / AdaLomo on a small torch model (the reference's model-based
optimizer tests, proj/tests/test_optim.cpp:220-316, with torch autograd as the tape)."""
import pytest

from paper_2312_00407_b200 import fused, optim
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def tiny_model(seed):
    g = torch.Generator().manual_seed(seed)
    m = torch.nn.Sequential(torch.nn.Embedding(17, 16), torch.nn.Linear(16, 24),
                            torch.nn.SiLU(), torch.nn.Linear(24, 17))
    with torch.no_grad():
        for p in m.parameters():
            p.copy_(torch.randn(p.shape, generator=g) * 0.2)
    return m.cuda()


IDS = torch.tensor([1, 4, 2, 9, 3, 7, 5, 0])
TGT = torch.tensor([4, 2, 9, 10, 7, 5, 0, 6])


def toy_loss(m):
    return torch.nn.functional.cross_entropy(m(IDS.cuda()), TGT.cuda())


def test_lomo_equals_stored_gradient_sgd():  # test_optim.cpp:220-246
    a, b = tiny_model(77), tiny_model(77)
    for _ in range(5):
        fused.lomo_fused_backward_step(list(a.parameters()), lambda: toy_loss(a), 0.05)
        b.zero_grad()
        toy_loss(b).backward()
        with torch.no_grad():
            for p in b.parameters():
                p -= 0.05 * p.grad
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.allclose(x, y, atol=1e-6)


def test_lomo_lr_zero_is_noop():  # test_optim.cpp:248-257
    m = tiny_model(5)
    snap = [p.detach().clone() for p in m.parameters()]
    fused.lomo_fused_backward_step(list(m.parameters()), lambda: toy_loss(m), 0.0)
    assert all(torch.equal(p, s) for p, s in zip(m.parameters(), snap))


def test_lomo_clip_matches_manually_clipped_sgd():  # test_optim.cpp:259-284
    a, b = tiny_model(13), tiny_model(13)
    fused.lomo_fused_backward_step(list(a.parameters()), lambda: toy_loss(a), 0.1,
                                   clip_norm=0.5)
    toy_loss(b).backward()
    norm2 = sum(float((p.grad.double() ** 2).sum()) for p in b.parameters())
    scale = min(1.0, 0.5 / norm2 ** 0.5)
    with torch.no_grad():
        for p in b.parameters():
            p -= (0.1 * scale) * p.grad
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.allclose(x, y, atol=1e-6)


def test_fused_steps_bound_live_gradients():  # test_optim.cpp:286-316
    """At every gradient-ready event only that parameter's gradient is alive: the fused
    hook drops each gradient right after its update, so the live gradient elements
    never exceed the largest tensor (the reference's RuntimeStats peak check)."""
    m = tiny_model(3)
    params = list(m.parameters())
    largest = max(p.numel() for p in params)
    peak = [0]

    def track(_p):  # registered first: runs before the fused hook of the same tensor
        peak[0] = max(peak[0], sum(q.grad.numel() for q in params if q.grad is not None))

    hs = [p.register_post_accumulate_grad_hook(track) for p in params]
    try:
        fused.lomo_fused_backward_step(params, lambda: toy_loss(m), 0.01)
        fused.lomo_fused_backward_step(params, lambda: toy_loss(m), 0.01, clip_norm=0.5)
        assert all(p.grad is None for p in params)
        st = optim.AdaLomoState(OptimizerConfig.defaults_for(Kind.ADALOMO),
                                [tuple(p.shape) for p in params])
        fused.adalomo_fused_step(params, lambda: toy_loss(m), 0.01, st)
        assert all(p.grad is None for p in params)
    finally:
        for h in hs:
            h.remove()
    assert 0 < peak[0] <= largest < sum(p.numel() for p in params)


class LoraLinear(torch.nn.Module):
    """y = x W^T + (x A^T) B^T * (alpha / r): frozen base W, trainable adapters A, B."""

    def __init__(self, base, r, seed):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.base = base
        self.base.weight.requires_grad_(False)
        if self.base.bias is not None:
            self.base.bias.requires_grad_(False)
        self.A = torch.nn.Parameter(torch.randn(r, base.in_features, generator=g) * 0.1)
        self.B = torch.nn.Parameter(torch.randn(base.out_features, r, generator=g) * 0.1)
        self.scale = 2.0 / r

    def forward(self, x):
        return self.base(x) + (x @ self.A.t()) @ self.B.t() * self.scale


def lora_model(seed, r=2):
    m = tiny_model(seed).cpu()
    m[0].weight.requires_grad_(False)
    m[1] = LoraLinear(m[1], r, seed + 1)
    m[3] = LoraLinear(m[3], r, seed + 2)
    return m.cuda()


def test_lomo_updates_adapters_only():  # test_lora.cpp:122-150
    m = lora_model(31)
    base = [p.detach().clone() for p in m.parameters() if not p.requires_grad]
    trainable = [p for p in m.parameters() if p.requires_grad]
    assert len(trainable) == 4 and base
    before = [p.detach().clone() for p in trainable]
    for _ in range(3):
        fused.lomo_fused_backward_step(trainable, lambda: toy_loss(m), 0.1)
    after = [p for p in m.parameters() if not p.requires_grad]
    assert all(torch.equal(x, y) for x, y in zip(after, base))  # bit-identical base
    assert sum(float((p.detach() - q).abs().sum()) for p, q in zip(trainable, before)) > 0


def test_state_scales_with_trainable_count():  # test_lora.cpp:152-163
    m = lora_model(31, r=2)
    trainable = sum(p.numel() for p in m.parameters() if p.requires_grad)
    total = sum(p.numel() for p in m.parameters())
    cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
    assert optim.FlatOptimizer(cfg, trainable, state_dtype="f64").state_bytes_runtime() == \
        2 * trainable * 8
    assert optim.FlatOptimizer(cfg, trainable).state_bytes_runtime() == 2 * trainable * 4
    assert trainable < total / 2


def test_adalomo_fused_equals_stored_gradient_apply_all():
    a, b = tiny_model(21), tiny_model(21)
    shapes = [tuple(p.shape) for p in a.parameters()]
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    sa, sb = optim.AdaLomoState(cfg, shapes), optim.AdaLomoState(cfg, shapes)
    for _ in range(3):
        fused.adalomo_fused_step(list(a.parameters()), lambda: toy_loss(a), 0.01, sa)
        b.zero_grad()
        toy_loss(b).backward()
        with torch.no_grad():
            for k, p in enumerate(b.parameters()):
                sb.apply(k, p.data, p.grad, 0.01)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)


@pytest.mark.parametrize("bucket", [None, 300, 1 << 20])
def test_bucketed_gradient_path_same_result(bucket):
    """Gradients packed into a flat bucket (the bucketed DP all-reduce path of f1) give
    the same bits as the per-parameter path; live gradients stay within the bucket."""
    a, b = tiny_model(8), tiny_model(8)
    for _ in range(3):
        fused.lomo_fused_backward_step(list(a.parameters()), lambda: toy_loss(a), 0.05,
                                       clip_norm=0.3)
        fused.lomo_fused_backward_step(list(b.parameters()), lambda: toy_loss(b), 0.05,
                                       clip_norm=0.3, bucket_elems=bucket)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)
    shapes = [tuple(p.shape) for p in a.parameters()]
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    sa, sb = optim.AdaLomoState(cfg, shapes), optim.AdaLomoState(cfg, shapes)
    fused.adalomo_fused_step(list(a.parameters()), lambda: toy_loss(a), 0.01, sa)
    fused.adalomo_fused_step(list(b.parameters()), lambda: toy_loss(b), 0.01, sb,
                             bucket_elems=bucket)
    for x, y in zip(a.parameters(), b.parameters()):
        assert torch.equal(x, y)
        assert x.grad is None and y.grad is None
