"""Golden vectors produced by the reference itself (tests/golden/make_golden.py over
oracle/_ref): the oracle restatement must reproduce them bit for bit (CPU), and the
GPU path must reproduce them bit for bit in f64 mode / within tolerance in fp32."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                         "reference_vectors.npz"))
FLAT = [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA]
ADA_SHAPES = [(6, 9), (7,), (33, 17)]
LR = 1e-3


def cfg_for(kind):
    c = OptimizerConfig.defaults_for(kind)
    c.weight_decay = 0.01
    c.update_interval = 2
    return c


@pytest.mark.parametrize("kind", FLAT)
def test_restatement_reproduces_reference_goldens(kind):
    o, p = O.OracleFlat(cfg_for(kind), G["flat_p0"].size), G["flat_p0"].copy()
    for t in range(1, 6):
        o.step(p, G[f"flat_g{t}"], LR)
    assert np.array_equal(p, G[f"{kind.name.lower()}_p"])
    for name, buf in o.state.items():
        assert np.array_equal(buf, G[f"{kind.name.lower()}_{name}"]), name


def test_restatement_lomo_clip_golden():
    p, g = G["lomo_p0"].copy(), G["lomo_g"]
    scale = O.orc.orc_clip_scale(O.orc.orc_sumsq_f64(O._ptr(np.ascontiguousarray(g)), g.size), 0.5)
    O.orc.orc_lomo_f64(O._ptr(p), O._ptr(np.ascontiguousarray(g)), p.size, 0.1, scale)
    np.testing.assert_allclose(p, G["lomo_clip_p"], rtol=0,
                               atol=4 * np.finfo(float).eps * np.abs(p).max())


def test_restatement_adalomo_golden():
    o = O.OracleAdaLomo(OptimizerConfig.defaults_for(Kind.ADALOMO), ADA_SHAPES)
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in ADA_SHAPES])])
    p = G["adalomo_p0"].copy()
    for t in range(1, 4):
        g = G[f"adalomo_g{t}"]
        for k in range(len(ADA_SHAPES)):
            pk = p[offs[k]:offs[k + 1]].copy()
            o.apply(k, pk, g[offs[k]:offs[k + 1]].copy(), 5e-3)
            p[offs[k]:offs[k + 1]] = pk
    assert np.array_equal(p, G["adalomo_p"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", FLAT)
def test_gpu_f64_mode_reproduces_reference_goldens(kind):
    import torch

    from paper_2312_00407_b200 import optim

    opt = optim.FlatOptimizer(cfg_for(kind), G["flat_p0"].size, state_dtype="f64")
    p = torch.from_numpy(G["flat_p0"].copy()).cuda()
    for t in range(1, 6):
        opt.step(p, torch.from_numpy(G[f"flat_g{t}"]).cuda(), LR)
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy(), G[f"{kind.name.lower()}_p"])
    for name, buf in opt.buffers():
        assert np.array_equal(buf.cpu().numpy(), G[f"{kind.name.lower()}_{name}"]), name


@pytest.mark.gpu
def test_gpu_adalomo_matches_reference_golden():
    import torch

    from paper_2312_00407_b200 import optim

    st = optim.AdaLomoState(OptimizerConfig.defaults_for(Kind.ADALOMO), ADA_SHAPES)
    p = torch.from_numpy(G["adalomo_p0"].astype(np.float32)).cuda()
    for t in range(1, 4):
        st.apply_all(p, torch.from_numpy(G[f"adalomo_g{t}"].astype(np.float32)).cuda(), 5e-3)
    torch.cuda.synchronize()
    want, got = G["adalomo_p"], p.cpu().numpy().astype(np.float64)
    rms = np.sqrt(np.mean(G["adalomo_p0"] ** 2))
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), rms)) <= 1e-5
