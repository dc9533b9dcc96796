"""Randomised parity sweep (fixed seed): random optimizer kind, length, element
offsets (alignment; the gradient's drawn apart from the parameters' in 40 % of the
cases), gradient dtype, hyper-parameters, step count and graph mode -- the
fp32 kernels must stay bit-exact with the restatement for every draw.
MCO_RANDOM_CASES=N / MCO_RANDOM_ADA_CASES=N widen the stored-state / AdaLomo sweeps
(defaults 40 / 12)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200 import optim
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

rng = np.random.default_rng(20260)
grng = np.random.default_rng(7)  # graph-mode draws (keeps the other draws unchanged)
orng = np.random.default_rng(11)  # gradient offsets apart from the parameters' (round 2)
CASES = []
for i in range(int(os.environ.get("MCO_RANDOM_CASES", "40"))):
    CASES.append(dict(kind=int(rng.integers(0, 4)), n=int(rng.choice([1, 7, 8, 9, 63, 4096,
                                                                       12345, 100003])),
                      off=int(rng.integers(0, 9)), bf16=bool(rng.random() < 0.3),
                      mixed=bool(rng.random() < 0.3), lr=float(10 ** rng.uniform(-5, -1)),
                      wd=float(rng.choice([0.0, 0.01, 0.1])), b1=float(rng.uniform(0.5, 0.99)),
                      b2=float(rng.uniform(0.9, 0.9999)), b3=float(rng.uniform(0.9, 0.999)),
                      k=int(rng.integers(1, 5)), steps=int(rng.integers(1, 5)), seed=i,
                      graph=bool(grng.random() < 0.3)))
    CASES[-1]["goff"] = int(orng.integers(0, 9)) if orng.random() < 0.4 else CASES[-1]["off"]


@pytest.mark.parametrize("c", CASES, ids=[f"case{i}" for i in range(len(CASES))])
def test_random_case_bit_exact(c):
    cfg = OptimizerConfig.defaults_for(Kind(c["kind"]))
    cfg.weight_decay, cfg.beta1, cfg.beta2, cfg.beta3 = c["wd"], c["b1"], c["b2"], c["b3"]
    cfg.update_interval = c["k"]
    n, off, goff = c["n"], c["off"], c["goff"]
    pbig = O.synth(n + off, c["seed"], 0, 0, 0, 0, -6, 0, False)
    tp = torch.from_numpy(pbig.copy()).cuda()
    p = pbig[off:].copy()
    opt, orc = optim.FlatOptimizer(cfg, n), O.OracleFlat(cfg, n, np.float32)
    if c["graph"]:  # device step counter + tabulated scalars (mco_flat_graph_enable)
        opt.enable_graph()
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda") if c["mixed"] else None
    for t in range(1, c["steps"] + 1):
        if c["bf16"]:
            gb = O.synth(n + goff, c["seed"], 1, 0, t, 0, -7, 10, False, "bf16")
            tg = torch.from_numpy(gb.view(np.int16)).cuda().view(torch.bfloat16)[goff:]
            g = O.bf16_to_f32(gb[goff:])
        else:
            gbig = O.synth(n + goff, c["seed"], 1, 0, t, 0, -7, 10, False)
            tg = torch.from_numpy(gbig).cuda()[goff:]
            g = gbig[goff:].copy()
        if out is not None:
            opt.step_mixed(tp[off:], tg, out, c["lr"])
        else:
            opt.step(tp[off:], tg, c["lr"])
        orc.step(p, np.ascontiguousarray(g), c["lr"])
    torch.cuda.synchronize()
    got = tp.cpu().numpy()
    assert np.array_equal(got[off:].view(np.uint32), p.view(np.uint32))
    assert np.array_equal(got[:off].view(np.uint32), pbig[:off].view(np.uint32))
    for name, buf in opt.buffers():
        assert np.array_equal(buf.cpu().numpy().view(np.uint32),
                              orc.state[name].view(np.uint32)), name
    if out is not None:
        assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16),
                              O.f32_to_bf16(p))


ADA_CASES = []
for i in range(int(os.environ.get("MCO_RANDOM_ADA_CASES", "12"))):
    shapes = []
    for _ in range(int(rng.integers(1, 6))):
        if rng.random() < 0.25:
            shapes.append((int(rng.integers(1, 3000)),))
        else:
            shapes.append((int(rng.integers(1, 300)), int(rng.choice([1, 3, 8, 17, 256, 1000,
                                                                      1032, 2100]))))
    ADA_CASES.append(dict(shapes=shapes, clip=float(rng.choice([0.0, 1e-3, 1e3])),
                          bf16=bool(rng.random() < 0.3), lr=float(10 ** rng.uniform(-4, -2)),
                          seed=100 + i))


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("c", ADA_CASES, ids=[f"ada{i}" for i in range(len(ADA_CASES))])
def test_random_adalomo_within_tolerance(c):
    shapes = c["shapes"]
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    clip = c["clip"] if c["clip"] > 0 else None
    ps = O.registry_params(shapes, c["seed"], np.float64)
    p0 = [x.copy() for x in ps]
    st, o = optim.AdaLomoState(cfg, shapes, grad_clip=clip), O.OracleAdaLomo(cfg, shapes)
    tp = torch.from_numpy(np.concatenate(ps).astype(np.float32)).cuda()
    for t in range(1, 3):
        gs = O.registry_grads(shapes, c["seed"], t, np.float32)
        gflat = np.concatenate(gs)
        if c["bf16"]:
            gb = O.f32_to_bf16(gflat)
            tg = torch.from_numpy(gb.view(np.int16)).cuda().view(torch.bfloat16)
            gflat = O.bf16_to_f32(gb)
        else:
            tg = torch.from_numpy(gflat).cuda()
        st.apply_all(tp, tg, c["lr"])
        g64 = gflat.astype(np.float64)
        scale = 1.0
        if c["clip"] > 0:
            scale = O.orc.orc_clip_scale(O.orc.orc_sumsq_f64(O._ptr(g64), g64.size), c["clip"])
        offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
        for k in range(len(shapes)):
            o.apply(k, ps[k], g64[offs[k]:offs[k + 1]].copy(), c["lr"], scale)
    torch.cuda.synchronize()
    got = tp.cpu().numpy().astype(np.float64)
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
    for k in range(len(shapes)):
        want = ps[k]
        rms = max(float(np.sqrt(np.mean(p0[k] ** 2))), 1e-30)
        err = np.max(np.abs(got[offs[k]:offs[k + 1]] - want) / np.maximum(np.abs(want), rms))
        assert err <= 1e-5, (k, shapes[k], err)
