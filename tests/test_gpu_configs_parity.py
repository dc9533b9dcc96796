"""Parity at BASELINE.json's stated sizes, through the C-ABI on the
GPU against the compiled reference (fp64), with the tests/parity.py bars:

* C1 exactly: configuration 1 (H=256, I=688, L=8, V=8192: 75 tensors, 10,522,880
  params), AdamW and Lion, fp32, 10 steps -- p, Δp and every state buffer within 1e-5
  of minicollie::optim::FlatOptimizer per element (test_optim.cpp:110-156's 100-step
  agreement, restated for fp32 storage), and bit-exact to the fp32 restatement (Lion's
  sign included).
* C3 on LLaMA-13B tensors: AdaLomo with the global grad-norm clip on the 13B shapes
  32000x5120 (embedding), 5120x5120, 13824x5120, 5120x13824 and a 5120 norm (357M
  params) -- the composed oracle (the reference's clip rule, optim.cpp:302-303, on the
  whole gradient, then the reference AdaLomoState::apply, optim.cpp:215-275).
"""
import numpy as np
import pytest

import oracle as O
import parity
from paper_2312_00407_b200 import optim, registry
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")]
torch = pytest.importorskip("torch")


def bits_equal(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


@pytest.mark.parametrize("kind", [Kind.ADAMW, Kind.LION])
def test_c1_config1_ten_steps_vs_reference(kind):
    shapes = registry.CONFIG1.shapes()
    P = registry.CONFIG1.param_count()
    assert P == 10_522_880 and len(shapes) == 75
    steps, lr = 10, 1e-3
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 1e-2
    p32 = np.concatenate(O.registry_params(shapes, registry.SEED, np.float32))
    p64, p0 = p32.astype(np.float64), p32.astype(np.float64)
    tp = torch.empty(P, device="cuda")
    registry.fill_params(tp, shapes)  # the device generator == the oracle's, bit for bit
    assert bits_equal(tp.cpu().numpy(), p32)
    tg = torch.empty(P, device="cuda")
    opt, r, o = optim.FlatOptimizer(cfg, P), O.RefFlat(cfg, P), O.OracleFlat(cfg, P, np.float32)
    for t in range(1, steps + 1):
        registry.fill_grads(tg, shapes, t)
        g = np.concatenate(O.registry_grads(shapes, registry.SEED, t, np.float32))
        opt.step(tp, tg, lr)
        r.step(p64, g.astype(np.float64), lr)
        o.step(p32, g, lr)
    torch.cuda.synchronize()
    got = tp.cpu().numpy()
    state = {nm: t.cpu().numpy() for nm, t in opt.buffers()}
    assert bits_equal(got, p32)  # the fp32 restatement (sign(0) = 0 for Lion)
    for nm, s in o.state.items():
        assert bits_equal(state[nm], s), nm
    e = parity.assert_flat_within(got, p64, p0, lr, steps, state, r.buffers(), kind.name)
    print(f"C1 {kind.name}: max errors vs the fp64 reference {e}")


def test_c3_adalomo_clip_on_13b_tensors_vs_reference():
    m = registry.LLAMA_13B
    H, I, V = m.hidden, m.intermediate, m.vocab
    shapes = [(V, H), (H,), (H, H), (I, H), (H, I)]
    n = sum(int(np.prod(s)) for s in shapes)
    steps, lr, clip = 2, 5e-4, 1.0
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ps = O.registry_params(shapes, registry.SEED, np.float64)
    p0 = np.concatenate(ps)
    tp = torch.from_numpy(p0.astype(np.float32)).cuda()
    st = optim.AdaLomoState(cfg, shapes, grad_clip=clip)
    r = O.RefAdaLomo(cfg, shapes)
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
    for t in range(1, steps + 1):
        gs = O.registry_grads(shapes, registry.SEED, t, np.float32)
        g = np.concatenate(gs)
        st.apply_all(tp, torch.from_numpy(g).cuda(), lr)
        g64 = g.astype(np.float64)
        scale = O.orc.orc_clip_scale(O.orc.orc_sumsq_f64(O._ptr(g64), g64.size), clip)
        assert scale < 1.0  # the clip is active on this set
        for k in range(len(shapes)):
            gk = np.ascontiguousarray(g64[offs[k]:offs[k + 1]] * scale)
            r.apply(k, ps[k], gk, lr)
    torch.cuda.synchronize()
    got = tp.cpu().numpy()
    want = np.concatenate(ps)
    e = parity.p_err(got, want, p0, lr)
    dp = parity.dp_err(got, want, p0, lr, steps)
    print(f"C3 AdaLomo+clip 13B tensors ({n} params): max p err {e.max():.3g}, "
          f"dp err {dp.max():.3g}")
    assert e.max() <= parity.TOL and dp.max() <= parity.TOL
