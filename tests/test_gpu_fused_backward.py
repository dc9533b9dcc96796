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
    m = tiny_model(3)
    params = list(m.parameters())
    live, peak = [0], [0]

    def track(p):
        live[0] += p.grad.numel()
        peak[0] = max(peak[0], live[0])

    hs = [p.register_post_accumulate_grad_hook(track) for p in params]
    fused.lomo_fused_backward_step(params, lambda: toy_loss(m), 0.01)
    for h in hs:
        h.remove()
    # hooks run in registration order per parameter: the fused hook drops the
    # gradient right after the update, so live gradients never exceed the largest
    largest = max(p.numel() for p in params)
    assert all(p.grad is None for p in params)
    st = optim.AdaLomoState(OptimizerConfig.defaults_for(Kind.ADALOMO),
                            [tuple(p.shape) for p in params])
    fused.adalomo_fused_step(params, lambda: toy_loss(m), 0.01, st)
    assert all(p.grad is None for p in params)
    assert largest > 0 and peak[0] <= sum(p.numel() for p in params)


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
