"""GPU parity of the fused optimizers (LOMO, AdaLomo) and the grad-norm reduction
through the C-ABI, against the oracle / compiled reference."""
import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200 import optim, registry
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                          np.ascontiguousarray(b).view(np.uint8))


# ---- LOMO ------------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 9, 100003, 1 << 22])
def test_lomo_f32_bf16_f64_bit_exact(n):
    p32 = O.synth(n, 4, 0, 0, 0, 0, -6, 0, False)
    g32 = O.synth(n, 4, 1, 0, 1, 0, -7, 10, False)
    t = dev(p32)
    optim.lomo_apply(t, dev(g32), 1e-2, 0.75)
    O.orc.orc_lomo_f32(O._ptr(p32), O._ptr(g32), n, 1e-2, 0.75)
    assert bits_equal(t.cpu().numpy(), p32)

    pb = O.synth(n, 4, 0, 0, 0, 0, -6, 0, False, "bf16")
    gb = O.synth(n, 4, 1, 0, 1, 0, -7, 10, False, "bf16")
    tb = dev(pb).view(torch.bfloat16)
    optim.lomo_apply(tb, dev(gb).view(torch.bfloat16), 1e-2, 1.0)
    O.orc.orc_lomo_bf16(O._ptr(pb), O._ptr(gb), n, 1e-2, 1.0)
    assert bits_equal(tb.view(torch.int16).cpu().numpy(), pb.view(np.int16))

    p64 = O.synth(n, 4, 0, 0, 0, 0, -6, 0, False, np.float64)
    g64 = O.synth(n, 4, 1, 0, 1, 0, -7, 10, False, np.float64)
    t64 = dev(p64)
    optim.lomo_apply(t64, dev(g64), 1e-2, 0.5)
    if O.ref is not None:  # the reference's lomo_apply itself
        O.ref_check(O.ref.ref_lomo_apply(O._ptr(p64), O._ptr(g64), n, 1e-2, 0.5))
    else:
        O.orc.orc_lomo_f64(O._ptr(p64), O._ptr(g64), n, 1e-2, 0.5)
    assert bits_equal(t64.cpu().numpy(), p64)


@pytest.mark.parametrize("dt", ["f32", "bf16", "f64"])
def test_sumsq_matches_oracle_and_is_deterministic(dt):
    n = 3 * (1 << 20) + 77
    if dt == "bf16":
        x = O.synth(n, 8, 1, 0, 1, 0, -7, 10, False, "bf16")
        want = O.orc.orc_sumsq_bf16(O._ptr(x), n)
        t = dev(x).view(torch.bfloat16)
    else:
        x = O.synth(n, 8, 1, 0, 1, 0, -7, 10, False, np.float32 if dt == "f32" else np.float64)
        want = (O.orc.orc_sumsq_f32 if dt == "f32" else O.orc.orc_sumsq_f64)(O._ptr(x), n)
        t = dev(x)
    a = optim.sumsq(t)
    b = optim.sumsq(t)
    optim.sumsq(t, out=b, accumulate=True)
    torch.cuda.synchronize()
    assert a.item() == pytest.approx(want, rel=1e-10)  # fp64 sums, different order
    assert bits_equal(np.array(a.item()), np.array(optim.sumsq(t).item()))
    assert b.item() == pytest.approx(2 * want, rel=1e-10)


@needs_ref
@pytest.mark.parametrize("clip", [None, 0.05, 1e9])
def test_lomo_clip_matches_reference_two_pass(clip):
    """lomo_fused_backward_step (optim.cpp:284-318, two backward passes) vs the flat
    form: one device sum-of-squares pass + the scaled update, in f64."""
    sizes = [4096, 17, 40000]
    ps = [O.synth(n, 5, 0, k, 0, 0, -6, 0, False, np.float64) for k, n in enumerate(sizes)]
    gs = [O.synth(n, 5, 1, k, 1, 0, -7, 10, False, np.float64) for k, n in enumerate(sizes)]
    tp, tg = dev(np.concatenate(ps)), dev(np.concatenate(gs))
    optim.lomo_step(tp, tg, 0.1, clip)
    O.ref_lomo_fused(ps, gs, 0.1, clip)
    torch.cuda.synchronize()
    want = np.concatenate(ps)
    # the reference sums g^2 in hook order, the device in a fixed tree: the clip
    # scale may differ in its last bit, i.e. each p by <= ~1 ulp of |p|_max
    np.testing.assert_allclose(tp.cpu().numpy(), want, rtol=0,
                               atol=4 * np.finfo(np.float64).eps * np.abs(want).max())


@pytest.mark.parametrize("variant", ["ldg", "tma", "tma_s3", "tma_s5"])
@pytest.mark.parametrize("n", [4096 + 3, 3 * 8192 + 17, (1 << 20) + 5])
def test_lomo_variants_bit_exact(variant, n):
    """The TMA LOMO pipeline (default) and the LDG kernel give the restatement's bits,
    fp32 and bf16, with and without the device-side clip scale."""
    prev = optim.flat_variant()
    optim.set_flat_variant(variant)
    try:
        for clip in (None, 0.01):
            p32 = O.synth(n, 6, 0, 0, 0, 0, -6, 0, False)
            g32 = O.synth(n, 6, 1, 0, 1, 0, -7, 10, False)
            t, tg = dev(p32), dev(g32)
            scale = 0.75
            if clip is None:
                optim.lomo_apply(t, tg, 1e-2, scale)
            else:
                s = optim.sumsq(tg)
                optim.lomo_apply_clipped(t, tg, 1e-2, s, clip)
                scale = O.orc.orc_clip_scale(float(s.item()), clip)
            O.orc.orc_lomo_f32(O._ptr(p32), O._ptr(g32), n, 1e-2, scale)
            assert bits_equal(t.cpu().numpy(), p32)

            pb = O.synth(n, 6, 0, 0, 0, 0, -6, 0, False, "bf16")
            gb = O.synth(n, 6, 1, 0, 1, 0, -7, 10, False, "bf16")
            tb, tgb = dev(pb).view(torch.bfloat16), dev(gb).view(torch.bfloat16)
            scale = 1.0
            if clip is None:
                optim.lomo_apply(tb, tgb, 1e-2, scale)
            else:
                s = optim.sumsq(tgb)
                optim.lomo_apply_clipped(tb, tgb, 1e-2, s, clip)
                scale = O.orc.orc_clip_scale(float(s.item()), clip)
            O.orc.orc_lomo_bf16(O._ptr(pb), O._ptr(gb), n, 1e-2, scale)
            assert bits_equal(tb.view(torch.int16).cpu().numpy(), pb.view(np.int16))
    finally:
        optim.set_flat_variant(prev)


def test_lomo_lr_zero_is_noop():  # test_optim.cpp:248-257
    p = O.synth(1000, 1, 0, 0, 0, 0, -6, 0, False)
    t = dev(p)
    optim.lomo_apply(t, dev(O.synth(1000, 1, 1, 0, 1, 0, -7, 0, False)), 0.0, 1.0)
    assert bits_equal(t.cpu().numpy(), p)


# ---- AdaLomo -----------------------------------------------------------------------------

SHAPES = [(6, 9), (7,), (3, 4), (33, 17), (64, 1040), (1, 5), (5, 1), (300, 256), (130,)]


def ada_inputs(shapes, steps, seed=9):
    ps = O.registry_params(shapes, seed, np.float64)
    gs = [O.registry_grads(shapes, seed, t, np.float64) for t in range(1, steps + 1)]
    return ps, gs


def ada_tol_ok(got32, want64, p0):
    rms = max(float(np.sqrt(np.mean(p0 ** 2))), 1e-30)
    err = np.abs(got32.astype(np.float64) - want64) / np.maximum(np.abs(want64), rms)
    return err.max() <= 1e-5, err.max()


@needs_ref
@pytest.mark.parametrize("form", ["hook", "all"])
def test_adalomo_matches_reference(form):
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    steps, lr = 4, 5e-3
    ps, gs = ada_inputs(SHAPES, steps)
    p0 = [p.copy() for p in ps]
    st = optim.AdaLomoState(cfg, SHAPES)
    r = O.RefAdaLomo(cfg, SHAPES)
    flat_p = dev(np.concatenate(ps).astype(np.float32))
    for t in range(steps):
        flat_g = dev(np.concatenate(gs[t]).astype(np.float32))
        if form == "all":
            st.apply_all(flat_p, flat_g, lr)
        else:
            for k in range(len(SHAPES)):
                a, b = int(st.offsets[k]), int(st.offsets[k + 1])
                st.apply(k, flat_p[a:b], flat_g[a:b], lr)
        for k in range(len(SHAPES)):
            r.apply(k, ps[k], gs[t][k], lr)
    torch.cuda.synchronize()
    got = flat_p.cpu().numpy()
    for k in range(len(SHAPES)):
        a, b = int(st.offsets[k]), int(st.offsets[k + 1])
        ok, e = ada_tol_ok(got[a:b], ps[k], p0[k])
        assert ok, (k, SHAPES[k], e)
        assert st.steps(k) == steps
    assert st.state_bytes_runtime() == r.state_bytes()


@needs_ref
def test_adalomo_state_matches_reference_state():
    """v_row / v_col / v_full after 3 steps vs the oracle's fp64 restatement."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ps, gs = ada_inputs(SHAPES, 3)
    st, o = optim.AdaLomoState(cfg, SHAPES), O.OracleAdaLomo(cfg, SHAPES)
    flat_p = dev(np.concatenate(ps).astype(np.float32))
    for t in range(3):
        st.apply_all(flat_p, dev(np.concatenate(gs[t]).astype(np.float32)), 1e-3)
        for k in range(len(SHAPES)):
            o.apply(k, ps[k], gs[t][k], 1e-3)
    torch.cuda.synchronize()
    for k, s in enumerate(SHAPES):
        e = o.entries[k]
        names = ("v_row", "v_col") if len(s) == 2 else ("v_full",)
        for nm in names:
            np.testing.assert_allclose(st.buffer(k, nm).cpu().numpy(), e[nm], rtol=2e-6,
                                       err_msg=f"{k} {nm}")


@needs_ref
@pytest.mark.parametrize("clip", [1e-3, 1e6])
def test_adalomo_global_clip_matches_composed_oracle(clip):
    """AdaLomo + global grad-norm clip (parity unpinned in the reference; composed
    oracle: the reference's clip rule, optim.cpp:302-303, scaling g, then the
    reference AdaLomoState::apply)."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ps, gs = ada_inputs(SHAPES, 2)
    p0 = [p.copy() for p in ps]
    st = optim.AdaLomoState(cfg, SHAPES, grad_clip=clip)
    o = O.OracleAdaLomo(cfg, SHAPES)
    flat_p = dev(np.concatenate(ps).astype(np.float32))
    for t in range(2):
        g = np.concatenate(gs[t]).astype(np.float32)
        st.apply_all(flat_p, dev(g), 1e-2)
        g64 = g.astype(np.float64)
        scale = O.orc.orc_clip_scale(O.orc.orc_sumsq_f64(O._ptr(g64), g64.size), clip)
        for k in range(len(SHAPES)):
            o.apply(k, ps[k], gs[t][k], 1e-2, scale)
    torch.cuda.synchronize()
    got = flat_p.cpu().numpy()
    for k in range(len(SHAPES)):
        a, b = int(st.offsets[k]), int(st.offsets[k + 1])
        ok, e = ada_tol_ok(got[a:b], ps[k], p0[k])
        assert ok, (k, e)


def test_adalomo_hook_form_with_device_norm_equals_all_form_clip():
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ps, gs = ada_inputs(SHAPES, 1)
    a, b = (optim.AdaLomoState(cfg, SHAPES, grad_clip=1e-3),
            optim.AdaLomoState(cfg, SHAPES, grad_clip=1e-3))
    fp = np.concatenate(ps).astype(np.float32)
    g = dev(np.concatenate(gs[0]).astype(np.float32))
    pa, pb = dev(fp), dev(fp)
    a.apply_all(pa, g, 1e-2)
    norm2 = optim.sumsq(g)
    for k in range(len(SHAPES)):
        s, e = int(b.offsets[k]), int(b.offsets[k + 1])
        b.apply(k, pb[s:e], g[s:e], 1e-2, grad_sumsq=norm2)
    torch.cuda.synchronize()
    np.testing.assert_allclose(pa.cpu().numpy(), pb.cpu().numpy(), rtol=1e-6, atol=1e-9)


def test_adalomo_rank1_exact():  # test_optim.cpp:318-352 through the GPU
    av, bv = np.array([0.5, -1.5, 2.0]), np.array([1.0, 0.25, -2.0, 0.5])
    g = np.outer(av, bv).ravel()
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    st = optim.AdaLomoState(cfg, [(3, 4)])
    p = torch.ones(12, device="cuda")
    st.apply(0, p, dev(g.astype(np.float32)), 0.01)
    delta = 1.0 - p.cpu().numpy().astype(np.float64)
    ratio = delta / (g / np.sqrt(g * g + cfg.eps))
    assert np.all(ratio > 0)
    np.testing.assert_allclose(ratio, ratio[0], rtol=1e-4)  # fp32 storage of p


def test_adalomo_bf16_grads_and_determinism():
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = registry.CONFIG1.shapes()[:12]
    n = sum(int(np.prod(s)) for s in shapes)
    outs = []
    for _ in range(2):
        st = optim.AdaLomoState(cfg, shapes)
        p = torch.empty(n, device="cuda")
        g = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        registry.fill_params(p, shapes)
        for t in (1, 2):
            registry.fill_grads(g, shapes, t)
            st.apply_all(p, g, 1e-3)
        outs.append(p.cpu().numpy())
    assert bits_equal(outs[0], outs[1])
    assert np.all(np.isfinite(outs[0]))


@pytest.mark.parametrize("clip", [None, 0.5])
def test_adalomo_bf16_params_round_the_f32_result(clip):
    """bf16 parameter storage (C5-style memory; fp32 arithmetic, RNE store): one step
    gives exactly RNE_bf16 of the fp32-parameter step on the same (bf16-valued) inputs,
    multi-tensor and hook forms; shapes include 1-D tensors and a column count that is
    not a multiple of 8 (scalar path)."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = registry.CONFIG1.shapes()[:10] + [(37, 29), (5,)]
    n = sum(int(np.prod(s)) for s in shapes)
    g = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    p32 = torch.empty(n, device="cuda")
    registry.fill_grads(g, shapes, 1)
    registry.fill_params(p32, shapes)
    p32 = p32.to(torch.bfloat16).float()  # bf16-representable starting point
    pb = p32.to(torch.bfloat16)
    qa, qb = p32.clone(), pb.clone()  # the hook form starts from the same point
    sa, sb = (optim.AdaLomoState(cfg, shapes, grad_clip=clip),
              optim.AdaLomoState(cfg, shapes, grad_clip=clip))
    sa.apply_all(p32, g, 1e-3)
    sb.apply_all(pb, g, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(p32.to(torch.bfloat16).view(torch.int16), pb.view(torch.int16))
    assert not torch.equal(pb.float(), p32)  # a real rounding happened somewhere
    if clip is None:  # hook form, one tensor at a time
        offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
        ha, hb = optim.AdaLomoState(cfg, shapes), optim.AdaLomoState(cfg, shapes)
        for k in reversed(range(len(shapes))):
            a, b = int(offs[k]), int(offs[k + 1])
            ha.apply(k, qa[a:b], g[a:b], 1e-3)
            hb.apply(k, qb[a:b], g[a:b], 1e-3)
        torch.cuda.synchronize()
        assert torch.equal(qa.to(torch.bfloat16).view(torch.int16), qb.view(torch.int16))


def test_adalomo_ignores_lomo_clip_threshold_like_the_reference():
    """cfg.clip_threshold is LOMO's field (optim.hpp:28); the reference's AdaLomoState
    never reads it (optim.cpp:215-275), so every AdaLomo form gives the same result with
    or without it; the global clip is the explicit grad_clip opt-in."""
    ps, gs = ada_inputs(SHAPES, 1)
    fp = np.concatenate(ps).astype(np.float32)
    g = dev(np.concatenate(gs[0]).astype(np.float32))
    outs = []
    for clip in (None, 1e-6):
        cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
        cfg.clip_threshold = clip
        st, tp = optim.AdaLomoState(cfg, SHAPES), dev(fp)
        st.apply_all(tp, g, 1e-2)
        outs.append(tp.cpu().numpy())
    assert bits_equal(outs[0], outs[1])
    st = optim.AdaLomoState(OptimizerConfig.defaults_for(Kind.ADALOMO), SHAPES)
    with pytest.raises(optim.ContractError, match="grad-norm clip is off"):
        st.apply(0, dev(fp)[:int(st.offsets[1])], g[:int(st.offsets[1])], 1e-2,
                 grad_sumsq=optim.sumsq(g))


def test_adalomo_rejects_bf16_params_with_f32_grads():
    st = optim.AdaLomoState(OptimizerConfig.defaults_for(Kind.ADALOMO), [(8, 8)])
    with pytest.raises(optim.ContractError, match="bf16 / bf16"):
        st.apply_all(torch.zeros(64, dtype=torch.bfloat16, device="cuda"),
                     torch.zeros(64, device="cuda"), 1e-3)


@needs_ref
def test_adalomo_config1_registry_vs_reference():
    """All 75 tensors of configuration 1 (10.5M params) through apply_all, 2 steps."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = registry.CONFIG1.shapes()
    n = registry.CONFIG1.param_count()
    st = optim.AdaLomoState(cfg, shapes)
    p = torch.empty(n, device="cuda")
    g = torch.empty(n, device="cuda")
    registry.fill_params(p, shapes)
    ps = O.registry_params(shapes, registry.SEED, np.float64)
    p0 = [x.copy() for x in ps]
    assert bits_equal(p.cpu().numpy(), np.concatenate(ps).astype(np.float32))
    r = O.RefAdaLomo(cfg, shapes)
    for t in (1, 2):
        registry.fill_grads(g, shapes, t)
        st.apply_all(p, g, 5e-4)
        gs = O.registry_grads(shapes, registry.SEED, t, np.float64)
        for k in range(len(shapes)):
            r.apply(k, ps[k], gs[k], 5e-4)
    torch.cuda.synchronize()
    got = p.cpu().numpy()
    for k in range(len(shapes)):
        a, b = int(st.offsets[k]), int(st.offsets[k + 1])
        ok, e = ada_tol_ok(got[a:b], ps[k], p0[k])
        assert ok, (k, shapes[k], e)


def test_lomo_host_path_equals_device_path():
    n = (1 << 24) + 999
    p = O.synth(n, 12, 0, 0, 0, 0, -6, 0, False)
    g = O.synth(n, 12, 1, 0, 1, 0, -7, 10, False)
    hp = p.copy()
    optim.lomo_apply(hp, g, 1e-2, 0.5)
    tp = dev(p)
    optim.lomo_apply(tp, dev(g), 1e-2, 0.5)
    torch.cuda.synchronize()
    assert bits_equal(hp, tp.cpu().numpy())
    # with the global-norm clip (two passes over the host gradient)
    hp2, tp2 = p.copy(), dev(p)
    optim.lomo_step(hp2, g, 1e-2, clip=0.1)
    optim.lomo_step(tp2, dev(g), 1e-2, clip=0.1)
    torch.cuda.synchronize()
    np.testing.assert_allclose(hp2, tp2.cpu().numpy(), rtol=0, atol=1e-9)


def test_lomo_host_clip_reuses_its_resident_gradient_buffer():
    """mco_lomo_apply_host keeps the device-resident gradient between calls (grown when a
    call needs more, freed by mco_host_release): every call -- smaller, larger, fp64
    (8 B gradients), after a release -- equals the device path."""
    import os
    for n, dt in [(1 << 22, np.float32), (1000, np.float32), ((1 << 23) + 5, np.float32),
                  ((1 << 22) + 3, np.float64), ("release", None), (1 << 21, np.float32)]:
        if n == "release":  # the 32 MiB buffer goes back to the driver
            before = torch.cuda.mem_get_info()[0]
            optim.host_release()
            if not os.environ.get("MCO_UNDER_SANITIZER"):  # (memcheck defers frees)
                assert torch.cuda.mem_get_info()[0] - before >= (16 << 20)
            continue
        p = O.synth(n, 12, 0, 0, 0, 0, -6, 0, False).astype(dt)
        g = O.synth(n, 12, 1, 0, 1, 0, -7, 10, False).astype(dt)
        hg, dg = g, torch.from_numpy(g).cuda()
        hp, tp = p.copy(), torch.from_numpy(p).cuda()
        optim.lomo_step(hp, hg, 1e-2, clip=0.1)
        optim.lomo_step(tp, dg, 1e-2, clip=0.1)
        torch.cuda.synchronize()
        assert bits_equal(hp, tp.cpu().numpy()), (n, dt)
    optim.host_release()


@pytest.mark.parametrize("clip", [None, 1e-3])
def test_adalomo_host_path_equals_device_path(clip):
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    ps, gs = ada_inputs(SHAPES, 2)
    a, b = (optim.AdaLomoState(cfg, SHAPES, grad_clip=clip),
            optim.AdaLomoState(cfg, SHAPES, grad_clip=clip))
    hp = np.concatenate(ps).astype(np.float32)
    tp = dev(hp)
    for t in range(2):
        g = np.concatenate(gs[t]).astype(np.float32)
        a.apply_all(hp, g, 1e-2)
        if clip is None:  # host path = per-tensor hook form
            for k in range(len(SHAPES)):
                s, e = int(b.offsets[k]), int(b.offsets[k + 1])
                b.apply(k, tp[s:e], dev(g[s:e]), 1e-2)
        else:
            b.apply_all(tp, dev(g), 1e-2)
    torch.cuda.synchronize()
    assert bits_equal(hp, tp.cpu().numpy())
    assert a.steps(0) == 2


def test_adalomo_list_form_equals_per_tensor():
    """mco_adalomo_apply_list (pointer table, > 64 tensors split in chunks) == one
    apply per tensor, bit for bit; misaligned / odd tensors included."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = registry.CONFIG1.shapes() + [(7, 13), (3,)]  # 77 tensors: two list chunks
    a = optim.AdaLomoState(cfg, shapes)
    b = optim.AdaLomoState(cfg, shapes)
    ps = [torch.randn(s, device="cuda") * 0.02 for s in shapes]
    qs = [p.clone() for p in ps]
    for t in range(2):
        gs = [torch.randn(s, device="cuda") * 1e-3 for s in shapes]
        for k in range(len(shapes)):
            a.apply(k, ps[k], gs[k], 1e-3)
        b.apply_list(0, qs, gs, 1e-3)
    torch.cuda.synchronize()
    for k in range(len(shapes)):
        assert torch.equal(ps[k], qs[k]), k
    assert [b.steps(k) for k in range(len(shapes))] == [2] * len(shapes)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_adalomo_mixed_alignment_call_equals_per_tensor(dt):
    """A multi-tensor call whose tensors disagree on the vector path (an odd-sized 1-D
    tensor shifts every later flat offset off the 8-element grid; a 13-column matrix
    never qualifies) runs the vector instance of each pass over the aligned tensors and
    the scalar instance over the rest: == one hook-form call per tensor, bit for bit."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = [(64, 256), (7,), (96, 512), (33, 13), (128, 1024), (5,), (40, 264), (300,)]
    n = sum(int(np.prod(s)) for s in shapes)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    p = (torch.randn(n, device="cuda") * 0.02).to(tdt)
    q = p.clone()
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
    a, b = optim.AdaLomoState(cfg, shapes), optim.AdaLomoState(cfg, shapes)
    for t in range(3):
        g = (torch.randn(n, device="cuda") * 1e-3).to(tdt)
        a.apply_all(p, g, 1e-3)
        for k in range(len(shapes)):
            lo, hi = int(offs[k]), int(offs[k + 1])
            b.apply(k, q[lo:hi], g[lo:hi], 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(p.view(torch.uint8), q.view(torch.uint8))


def test_adalomo_and_lomo_replay_from_a_cuda_graph():
    """AdaLomo's chain (step counter, scalars and clip scale on the device, PDL launches)
    and LOMO capture into a CUDA graph: three replays == three eager steps, bit for bit,
    and the step counter counts the replays."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = registry.CONFIG1.shapes()[:12]
    n = sum(int(np.prod(s)) for s in shapes)
    p = torch.empty(n, device="cuda")
    g = torch.empty(n, device="cuda")
    registry.fill_params(p, shapes)
    registry.fill_grads(g, shapes, 1)
    pe, pg = p.clone(), p.clone()
    qe, qg = p.clone(), p.clone()
    se, sg = optim.AdaLomoState(cfg, shapes), optim.AdaLomoState(cfg, shapes)
    for _ in range(3):
        se.apply_all(pe, g, 1e-3)
        optim.lomo_apply(qe, g, 1e-3, 0.5)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        sg.apply_all(pg, g, 1e-3)
        optim.lomo_apply(qg, g, 1e-3, 0.5)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(pe, pg)
    assert torch.equal(qe, qg)
    assert [sg.steps(k) for k in range(len(shapes))] == [3] * len(shapes)


def test_adalomo_hook_form_replays_from_a_cuda_graph():
    """The per-tensor hook form (PDL chains, the early-started next K1, the one-launch
    cluster kernel of small 1-D tensors) captured on a side stream: three replays ==
    three eager rounds of hook calls, bit for bit."""
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    shapes = registry.CONFIG1.shapes()[:12]
    n = sum(int(np.prod(s)) for s in shapes)
    offs = np.concatenate([[0], np.cumsum([int(np.prod(s)) for s in shapes])])
    p = torch.empty(n, device="cuda")
    g = torch.empty(n, device="cuda")
    registry.fill_params(p, shapes)
    registry.fill_grads(g, shapes, 1)
    pe, pg = p.clone(), p.clone()
    se, sg = optim.AdaLomoState(cfg, shapes), optim.AdaLomoState(cfg, shapes)
    s = torch.cuda.Stream()

    def hooks(st, q):
        for k in reversed(range(len(shapes))):
            a, b = int(offs[k]), int(offs[k + 1])
            st.apply(k, q[a:b], g[a:b], 1e-3, stream=s)

    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for _ in range(3):
            hooks(se, pe)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        hooks(sg, pg)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(pe, pg)
    assert [sg.steps(k) for k in range(len(shapes))] == [3] * len(shapes)


@pytest.mark.parametrize("dt", ["f32", "bf16", "f32_bf16g", "f64"])
@pytest.mark.parametrize("clip", [None, 0.5])
def test_lomo_apply_list_equals_per_tensor(dt, clip):
    """mco_lomo_apply_list (one launch per 40 tensors, odd / tiny / empty / unaligned
    tensors) == lomo_apply / lomo_apply_clipped per tensor, bit for bit."""
    pdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f32_bf16g": torch.float32,
           "f64": torch.float64}[dt]
    gdt = torch.bfloat16 if dt in ("bf16", "f32_bf16g") else pdt
    gen = torch.Generator(device="cuda").manual_seed(3)
    sizes = [4096, 7, 0, 1000, 65536, 3, 12288, 1] * 6  # 48 tensors: two launches
    base = [torch.randn(n + 1, generator=gen, device="cuda", dtype=torch.float32) for n in sizes]
    # every third tensor starts one element in: unaligned views take the scalar path
    ps = [(b[1:] if k % 3 == 2 else b[:-1]).to(pdt) for k, b in enumerate(base)]
    ps = [p if p.is_contiguous() else p.contiguous() for p in ps]
    gs = [(torch.randn(n, generator=gen, device="cuda") * 0.1).to(gdt) for n in sizes]
    qs = [p.clone() for p in ps]
    norm2 = None
    if clip is not None:
        norm2 = torch.zeros((), dtype=torch.float64, device="cuda")
        for g in gs:
            optim.sumsq(g, out=norm2, accumulate=True)
    optim.lomo_apply_list(ps, gs, 1e-2, 1.0, norm2, clip)
    for q, g in zip(qs, gs):
        if clip is None:
            optim.lomo_apply(q, g, 1e-2, 1.0)
        else:
            optim.lomo_apply_clipped(q, g, 1e-2, norm2, clip)
    torch.cuda.synchronize()
    for p, q in zip(ps, qs):
        assert torch.equal(p, q)


K6_CHILD = r"""
import hashlib, sys
import torch
sys.path.insert(0, sys.argv[1])
from paper_2312_00407_b200 import optim, registry
from paper_2312_00407_b200.optim import Kind, OptimizerConfig
cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
shapes = registry.CONFIG1.shapes()[:12]
n = sum(int(torch.tensor(s).prod()) for s in shapes)
h = hashlib.sha256()
for pdt, gdt in ((torch.float32, torch.float32), (torch.float32, torch.bfloat16),
                 (torch.bfloat16, torch.bfloat16)):
    p = torch.empty(n, device="cuda")
    registry.fill_params(p, shapes)
    p = p.to(pdt)
    g = torch.empty(n, device="cuda")
    registry.fill_grads(g, shapes, 1)
    g = g.to(gdt)
    st = optim.AdaLomoState(cfg, shapes)
    st.apply_all(p, g, 1e-3)
    q = p.clone()
    offs = [0]
    for s in shapes:
        offs.append(offs[-1] + int(torch.tensor(s).prod()))
    for k in range(len(shapes)):
        st.apply(k, q[offs[k]:offs[k + 1]], g[offs[k]:offs[k + 1]], 1e-3)
    torch.cuda.synchronize()
    h.update(p.view(torch.uint8).cpu().numpy().tobytes())
    h.update(q.view(torch.uint8).cpu().numpy().tobytes())
print(h.hexdigest())
"""


def test_adalomo_k6_traversals_bit_identical():
    """K6's three traversals (tiles, flat chunks, the cp.async.bulk pipeline; the
    MCO_ADALOMO_K6 A/B knob, read once per process) give the same bits, multi-tensor and
    hook forms, every (params, grads) dtype pair."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("tiles", "chunks", "tma"):
        r = subprocess.run([sys.executable, "-c", K6_CHILD, root], capture_output=True,
                           text=True, timeout=600, env=dict(os.environ, MCO_ADALOMO_K6=v))
        assert r.returncode == 0, r.stderr[-2000:]
        out[v] = r.stdout.strip().splitlines()[-1]
    assert len(set(out.values())) == 1, out
