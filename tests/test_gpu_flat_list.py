"""FlatOptimizer list form (mco_flat_step_list): separate parameter / gradient tensors
over the flat state.  Bar: bit-identical to FlatOptimizer::step (optim.cpp:100-112)
over the concatenated vector -- parameters and every state buffer -- for every kind and
dtype mode, with odd / empty / unaligned tensors, more tensors than one launch carries,
and in graph mode."""
import os

import pytest

from paper_2312_00407_b200 import optim
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

KINDS = [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA]
# odd sizes shift every later state offset off the 8-element grid (scalar path for
# those tensors), zeros are skipped, the large ones run the vector path
SIZES = [4096, 1000, 7, 0, 65536, 3, 12288, 1, 262144, 4104, 0, 9999]


def _cfg(kind):
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 0.01
    if kind == Kind.SOPHIA:
        cfg.update_interval = 2
    return cfg


def _tensors(sizes, pdt, gdt, seed=5, steps=3):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    ps = [torch.randn(n, generator=gen, device="cuda", dtype=pdt) * 0.02 for n in sizes]
    gs = [[(torch.randn(n, generator=gen, device="cuda", dtype=pdt) * 1e-2).to(gdt)
           for n in sizes] for _ in range(steps)]
    return ps, gs


def _check_equal(flat_opt, flat_p, list_opt, ps):
    assert torch.equal(torch.cat([p.reshape(-1) for p in ps]), flat_p)
    for (na, a), (nb, b) in zip(flat_opt.buffers(), list_opt.buffers()):
        assert na == nb and torch.equal(a, b), na


@pytest.mark.parametrize("kind", KINDS, ids=lambda k: k.name.lower())
@pytest.mark.parametrize("mode", ["f32", "bf16g", "f64"])
def test_list_equals_flat_step_over_the_concatenation(kind, mode):
    cfg = _cfg(kind)
    pdt = torch.float64 if mode == "f64" else torch.float32
    gdt = torch.bfloat16 if mode == "bf16g" else pdt
    sd = "f64" if mode == "f64" else "f32"
    ps, gs = _tensors(SIZES, pdt, gdt)
    total = sum(SIZES)
    flat = optim.FlatOptimizer(cfg, total, state_dtype=sd)
    lst = optim.FlatOptimizer(cfg, total, state_dtype=sd)
    flat_p = torch.cat([p.reshape(-1) for p in ps])
    for t, g in enumerate(gs):
        lr = 1e-3 * (1 + t)
        flat.step(flat_p, torch.cat([x.reshape(-1) for x in g]), lr)
        lst.step_list(ps, g, lr)
    torch.cuda.synchronize()
    _check_equal(flat, flat_p, lst, ps)
    assert lst.steps_taken() == len(gs)


def test_list_more_tensors_than_one_launch_and_2d_views():
    cfg = _cfg(Kind.ADAMW)
    sizes = [(64, 48)] * 50 + [(128, 40)] * 47 + [(5, 3)] * 10  # 107 tensors, 3 launches
    gen = torch.Generator(device="cuda").manual_seed(1)
    ps = [torch.randn(*s, generator=gen, device="cuda") for s in sizes]
    total = sum(p.numel() for p in ps)
    flat = optim.FlatOptimizer(cfg, total + 100)  # owned state may be larger
    lst = optim.FlatOptimizer(cfg, total + 100)
    flat_p = torch.cat([p.reshape(-1) for p in ps])
    for t in range(2):
        g = [torch.randn(*s, generator=gen, device="cuda") for s in sizes]
        flat.step(flat_p, torch.cat([x.reshape(-1) for x in g]), 1e-3)
        lst.step_list(ps, g, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([p.reshape(-1) for p in ps]), flat_p)
    for (_, a), (_, b) in zip(flat.buffers(), lst.buffers()):
        assert torch.equal(a[:total], b[:total])


@pytest.mark.parametrize("kind", [Kind.ADAN, Kind.SOPHIA], ids=lambda k: k.name.lower())
def test_list_replays_from_a_cuda_graph(kind):
    cfg = _cfg(kind)
    ps, gs = _tensors(SIZES, torch.float32, torch.float32, steps=4)
    total = sum(SIZES)
    eager = optim.FlatOptimizer(cfg, total)
    graphed = optim.FlatOptimizer(cfg, total)
    pe = [p.clone() for p in ps]
    for t, g in enumerate(gs):
        eager.step_list(pe, g, 1e-3 / (1 + t))
    lr_t = torch.zeros((), dtype=torch.float64, device="cuda")
    g_static = [torch.empty_like(x) for x in gs[0]]
    graphed.enable_graph(lr_t)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        graphed.step_list(ps, g_static, 0.0)
    for t, g in enumerate(gs):
        for d, s in zip(g_static, g):
            d.copy_(s)
        lr_t.fill_(1e-3 / (1 + t))
        graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(pe, ps):
        assert torch.equal(a, b)
    assert graphed.steps_taken() == len(gs)


def test_list_contract_errors():
    cfg = _cfg(Kind.ADAMW)
    opt = optim.FlatOptimizer(cfg, 10)
    a = torch.zeros(6, device="cuda")
    with pytest.raises(optim.ContractError, match="exceed"):
        opt.step_list([a, a.clone()], [a.clone(), a.clone()], 1e-3)
    with pytest.raises(optim.ContractError, match="mixed dtypes"):
        opt.step_list([a[:2], a[2:4]], [a[:2].clone(), a[2:4].bfloat16()], 1e-3)
    with pytest.raises(optim.ContractError, match="length mismatch"):
        opt.step_list([a], [], 1e-3)
    opt.step_list([], [], 1e-3)  # an empty list still counts as a step
    assert opt.steps_taken() == 1


@pytest.mark.parametrize("seed", range(int(os.environ.get("MCO_LIST_CASES", "12"))))
def test_list_randomised_sweep(seed):
    """Random kinds, dtype modes, tensor counts (1-90: up to three launches), sizes
    (odd, tiny, vector-sized, empty), step counts and graph mode: list == flat, bit for
    bit.  MCO_LIST_CASES=N widens the sweep (default 12)."""
    import random

    rnd = random.Random(seed)
    kind = rnd.choice(KINDS)
    mode = rnd.choice(["f32", "bf16g", "f64"])
    cfg = _cfg(kind)
    cfg.weight_decay = rnd.choice([0.0, 0.01, 0.1])
    pdt = torch.float64 if mode == "f64" else torch.float32
    gdt = torch.bfloat16 if mode == "bf16g" else pdt
    sd = "f64" if mode == "f64" else "f32"
    sizes = [rnd.choice([0, 1, 3, 8, 17, 256, 1000, 4096, 8200, 40000])
             for _ in range(rnd.randint(1, 90))]
    steps = rnd.randint(1, 4)
    ps, gs = _tensors(sizes, pdt, gdt, seed=seed, steps=steps)
    total = sum(sizes)
    flat = optim.FlatOptimizer(cfg, max(total, 1), state_dtype=sd)
    lst = optim.FlatOptimizer(cfg, max(total, 1), state_dtype=sd)
    if rnd.random() < 0.3:
        lst.enable_graph()  # eager calls on the device step counter
    flat_p = torch.cat([p.reshape(-1) for p in ps])
    for t, g in enumerate(gs):
        lr = rnd.choice([1e-4, 1e-3, 3e-2])
        flat.step(flat_p, torch.cat([x.reshape(-1) for x in g]), lr)
        lst.step_list(ps, g, lr)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([p.reshape(-1) for p in ps]), flat_p)
    for (na, a), (nb, b) in zip(flat.buffers(), lst.buffers()):
        assert na == nb and torch.equal(a[:total], b[:total]), na
