"""Parity at BASELINE.json's full size: the whole LLaMA-7B-shaped set (6,738,415,616
params, 291 tensors, flat buffers of 27 GB: element offsets above 2^32) through the
product path, checked tensor by tensor on the CPU for a sample of tensors that the
counter-based generator regenerates exactly (first, middle, the 1-D norms, and the
last tensor, which starts at element 6.6e9).

* Adan (all four stored state buffers, the dominant kernel) -- bit-exact vs the fp32
  restatement, p and every state buffer, over two steps (t == 1 skips g_prev);
* AdaLomo (no clip: tensors are independent) -- within the fp32 tolerance of the fp64
  restatement."""
import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200 import optim, registry
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SHAPES = registry.LLAMA_7B.shapes()
OFFS = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in SHAPES])])
SAMPLE = [0, 1, 137, 146, len(SHAPES) - 2, len(SHAPES) - 1]  # embed, norm, mid q/down, last


def _tensor_p(k, dtype):
    return O.registry_params([SHAPES[k]], registry.SEED, dtype)[0] if len(SHAPES[k]) == 1 \
        else O.synth(int(OFFS[k + 1] - OFFS[k]), registry.SEED, 0, k, 0, SHAPES[k][1], -6, 0,
                     False, dtype)


def _tensor_g(k, step, dtype):
    s = SHAPES[k]
    n = int(OFFS[k + 1] - OFFS[k])
    if len(s) == 2:
        return O.synth(n, registry.SEED, 1, k, step, s[1], -7, 10, True, dtype)
    return O.synth(n, registry.SEED, 1, k, step, 0, -7, 10, False, dtype)


@pytest.fixture(scope="module")
def flat_set():
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")
    P = int(OFFS[-1])
    assert P == registry.LLAMA_7B.param_count() == 6738415616
    p = torch.empty(P, device="cuda")
    g = torch.empty(P, device="cuda")
    yield p, g
    del p, g
    torch.cuda.empty_cache()


def test_adan_full_7b_bit_exact_sampled(flat_set):
    p, g = flat_set
    registry.fill_params(p, SHAPES)
    cfg = OptimizerConfig.defaults_for(Kind.ADAN)
    cfg.weight_decay = 0.02
    opt = optim.FlatOptimizer(cfg, p.numel())
    assert OFFS[SAMPLE[-1]] > (1 << 32)
    for t in (1, 2):
        registry.fill_grads(g, SHAPES, t)
        opt.step(p, g, 5e-5)
    torch.cuda.synchronize()
    bufs = dict(opt.buffers())
    for k in SAMPLE:
        a, b = int(OFFS[k]), int(OFFS[k + 1])
        want = _tensor_p(k, np.float32)
        orc = O.OracleFlat(cfg, b - a, np.float32)
        for t in (1, 2):
            orc.step(want, _tensor_g(k, t, np.float32), 5e-5)
        assert np.array_equal(p[a:b].cpu().numpy().view(np.uint32), want.view(np.uint32)), k
        for name, buf in orc.state.items():
            got = bufs[name][a:b].cpu().numpy()
            assert np.array_equal(got.view(np.uint32), buf.view(np.uint32)), (k, name)
    del opt, bufs


def test_adalomo_full_7b_sampled(flat_set):
    p, g = flat_set
    registry.fill_params(p, SHAPES)
    registry.fill_grads(g, SHAPES, 1)
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    st = optim.AdaLomoState(cfg, SHAPES)
    st.apply_all(p, g, 5e-4)
    torch.cuda.synchronize()
    for k in SAMPLE:
        a, b = int(OFFS[k]), int(OFFS[k + 1])
        want = _tensor_p(k, np.float64)
        p0 = want.copy()
        O.OracleAdaLomo(cfg, [SHAPES[k]]).apply(0, want, _tensor_g(k, 1, np.float64), 5e-4)
        got = p[a:b].cpu().numpy().astype(np.float64)
        rms = float(np.sqrt(np.mean(p0 ** 2)))
        err = np.max(np.abs(got - want) / np.maximum(np.abs(want), rms))
        assert err <= 1e-5, (k, err)
        assert not np.array_equal(got, p0)  # the step moved the tensor
