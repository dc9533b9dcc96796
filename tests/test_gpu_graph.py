"""FlatOptimizer graph mode (mco_flat_graph_enable): a step captured into a CUDA graph
replays as the next step -- the step counter and the step scalars live on the device
(flat_graph_prep, flat.cu).  The bar is bit-identity with eager steps
(FlatOptimizer::step, optim.cpp:100-112) over a learning-rate schedule, for every kind,
dtype mode and alignment phase, past the end of the scalar table, and across
disable / enable."""
import numpy as np
import pytest

from paper_2312_00407_b200 import optim
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

N = 100_003  # odd: TMA body + LDG tail
STEPS = 7
KINDS = [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA]


def _cfg(kind):
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 0.01
    if kind == Kind.SOPHIA:
        cfg.update_interval = 3  # refresh at t = 1, 4, 7
    return cfg


def _inputs(mode, phase):
    gen = torch.Generator(device="cuda").manual_seed(7)
    pdt = torch.float64 if mode == "f64" else torch.float32
    gdt = torch.bfloat16 if mode in ("bf16g", "mixed") else pdt
    base = torch.randn(N + 8, generator=gen, device="cuda", dtype=pdt)
    grads = [torch.randn(N, generator=gen, device="cuda", dtype=pdt).to(gdt) * 0.1
             for _ in range(STEPS)]
    return base, grads, phase


def _lrs():
    return [1e-3 * 0.8 ** i for i in range(STEPS)]


def _view(buf, phase):
    return buf[phase:phase + N]


@pytest.mark.parametrize("kind", KINDS, ids=lambda k: k.name.lower())
@pytest.mark.parametrize("mode", ["f32", "bf16g", "mixed", "f64"])
@pytest.mark.parametrize("phase", [0, 3])
def test_graph_replays_equal_eager_steps(kind, mode, phase):
    cfg = _cfg(kind)
    sd = "f64" if mode == "f64" else "f32"
    base, grads, _ = _inputs(mode, phase)
    eager = optim.FlatOptimizer(cfg, N, state_dtype=sd)
    graphed = optim.FlatOptimizer(cfg, N, state_dtype=sd)
    pe_buf, pg_buf = base.clone(), base.clone()
    pe, pg = _view(pe_buf, phase), _view(pg_buf, phase)
    oe = torch.zeros(N, dtype=torch.bfloat16, device="cuda")
    og = oe.clone()
    for i, lr in enumerate(_lrs()):
        if mode == "mixed":
            eager.step_mixed(pe, grads[i], oe, lr)
        else:
            eager.step(pe, grads[i], lr)

    lr_t = torch.zeros((), dtype=torch.float64, device="cuda")
    g_static = torch.empty_like(grads[0])
    graphed.enable_graph(lr_t)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        if mode == "mixed":
            graphed.step_mixed(pg, g_static, og, 0.0)
        else:
            graphed.step(pg, g_static, 0.0)  # lr comes from lr_t
    assert graphed.steps_taken() == 0  # capture does not run the step
    for i, lr in enumerate(_lrs()):
        g_static.copy_(grads[i])
        lr_t.fill_(lr)
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(pe_buf, pg_buf)
    if mode == "mixed":
        assert torch.equal(oe, og)
    assert graphed.steps_taken() == STEPS
    for (na, a), (nb, b) in zip(eager.buffers(), graphed.buffers()):
        assert na == nb and torch.equal(a, b), na


@pytest.mark.parametrize("kind", KINDS, ids=lambda k: k.name.lower())
@pytest.mark.parametrize("start", [100, 50_000, 10_000_000])
def test_graph_mode_at_late_steps(kind, start):
    """Past the end of the scalar table (1 - beta^t has rounded to 1.0) and deep inside
    it: graph-mode steps (eager calls, no capture) == host-scalar steps."""
    cfg = _cfg(kind)
    base, grads, _ = _inputs("f32", 0)
    a = optim.FlatOptimizer(cfg, N)
    b = optim.FlatOptimizer(cfg, N)
    a.set_steps_taken(start)
    b.enable_graph()
    b.set_steps_taken(start)
    pa, pb = base[:N].clone(), base[:N].clone()
    for i, lr in enumerate(_lrs()[:4]):
        a.step(pa, grads[i], lr)
        b.step(pb, grads[i], lr)
    assert torch.equal(pa, pb)
    assert b.steps_taken() == start + 4


def test_graph_disable_and_reenable_keep_the_step_count():
    cfg = _cfg(Kind.ADAN)
    base, grads, _ = _inputs("f32", 0)
    a = optim.FlatOptimizer(cfg, N)
    b = optim.FlatOptimizer(cfg, N)
    pa, pb = base[:N].clone(), base[:N].clone()
    for i, lr in enumerate(_lrs()):
        a.step(pa, grads[i], lr)
        if i == 2:
            b.enable_graph()
        if i == 5:
            b.disable_graph()
            assert b.steps_taken() == 5
            b.enable_graph()
        b.step(pb, grads[i], lr)
    assert torch.equal(pa, pb)
    b.disable_graph()
    assert b.steps_taken() == STEPS


def test_graph_mode_refuses_host_span_steps():
    cfg = _cfg(Kind.ADAMW)
    opt = optim.FlatOptimizer(cfg, 64)
    opt.enable_graph()
    p = np.zeros(64, np.float32)
    with pytest.raises(optim.ContractError, match="graph mode"):
        opt.step(p, p.copy(), 1e-3)
    with pytest.raises(optim.ContractError):
        opt.enable_graph(torch.zeros((), dtype=torch.float32, device="cuda"))
