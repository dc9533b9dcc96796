"""Pin the oracle (CPU, no GPU): the plain-C restatement against the reference
itself (oracle/_ref, compiled from /root/reference) and against the
reference's own known-answer tests (proj/tests/test_optim.cpp)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")

FLAT_KINDS = [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA]


def cfg_for(kind, **kw):
    c = OptimizerConfig.defaults_for(kind)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def grads(n, step, seed=7, dtype=np.float64):
    return O.synth(n, seed, 1, 3, step, 0, -3, 6, False, dtype)


# ---- restatement f64 == reference, bit for bit -------------------------------------------

@needs_ref
@pytest.mark.parametrize("kind", FLAT_KINDS)
@pytest.mark.parametrize("n", [1, 7, 1000])
def test_restatement_f64_bit_exact_vs_reference(kind, n):
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=3)
    p_ref = O.synth(n, 1, 0, 0, 0, 0, -1, 0, False, np.float64)
    p_orc = p_ref.copy()
    r, o = O.RefFlat(cfg, n), O.OracleFlat(cfg, n, np.float64)
    for t in range(1, 26):
        g = grads(n, t)
        r.step(p_ref, g, 1e-3)
        o.step(p_orc, g, 1e-3)
    assert np.array_equal(p_ref.view(np.uint64), p_orc.view(np.uint64))
    rb = r.buffers()
    assert list(rb) == list(o.state)  # same names, same order (optim.cpp:173-181)
    for name in rb:
        assert np.array_equal(rb[name].view(np.uint64), o.state[name].view(np.uint64)), name
    assert r.steps() == o.t == 25


@needs_ref
def test_restatement_lomo_bit_exact_vs_reference():
    n = 4099
    p_ref = O.synth(n, 3, 0, 0, 0, 0, 0, 0, False, np.float64)
    p_orc = p_ref.copy()
    g = grads(n, 1)
    O.ref_check(O.ref.ref_lomo_apply(O._ptr(p_ref), O._ptr(g), n, 0.05, 0.7))
    O.orc.orc_lomo_f64(O._ptr(p_orc), O._ptr(g), n, 0.05, 0.7)
    assert np.array_equal(p_ref, p_orc)


@needs_ref
@pytest.mark.parametrize("clip", [None, 0.5, 1e9])
def test_restatement_lomo_clip_vs_reference_two_pass(clip):
    """optim.cpp:284-318 (two backward passes) == one sum-of-squares pass + update."""
    sizes = [17, 256, 5]
    ps = [O.synth(n, 5, 0, k, 0, 0, 0, 0, False, np.float64) for k, n in enumerate(sizes)]
    gs = [O.synth(n, 5, 1, k, 1, 0, -1, 0, False, np.float64) for k, n in enumerate(sizes)]
    ref_ps = [p.copy() for p in ps]
    O.ref_lomo_fused(ref_ps, gs, 0.1, clip)
    allg = np.concatenate(gs)
    scale = 1.0 if clip is None else O.orc.orc_clip_scale(O.orc.orc_sumsq_f64(O._ptr(allg),
                                                                               allg.size), clip)
    for p, g, rp in zip(ps, gs, ref_ps):
        O.orc.orc_lomo_f64(O._ptr(p), O._ptr(g), p.size, 0.1, scale)
        # sum order over tensors follows hook order in the reference: <= a few ulp
        np.testing.assert_allclose(p, rp, rtol=1e-14, atol=0)


ADA_SHAPES = [(6, 9), (7,), (3, 4), (33, 17), (1, 5), (5, 1)]


@needs_ref
def test_restatement_adalomo_bit_exact_vs_reference():
    cfg = cfg_for(Kind.ADALOMO)
    r, o = O.RefAdaLomo(cfg, ADA_SHAPES), O.OracleAdaLomo(cfg, ADA_SHAPES)
    ps = [O.synth(int(np.prod(s)), 9, 0, k, 0, 0, -2, 0, False, np.float64)
          for k, s in enumerate(ADA_SHAPES)]
    ps_o = [p.copy() for p in ps]
    for t in range(1, 6):
        for k, s in enumerate(ADA_SHAPES):
            g = O.synth(int(np.prod(s)), 9, 1, k, t, 0, -4, 3, False, np.float64)
            r.apply(k, ps[k], g, 0.01)
            o.apply(k, ps_o[k], g, 0.01)
    for a, b in zip(ps, ps_o):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert r.state_bytes() == sum((s[0] + s[1]) * 8 if len(s) == 2 else s[0] * 8
                                  for s in ADA_SHAPES)


@needs_ref
@pytest.mark.parametrize("P,N", [(10, 4), (10, 3), (10, 1), (7, 8), (0, 2), (10522880, 8),
                                 (6738415616, 8), (65285660672, 3)])
def test_zero_plan_three_ways(P, N):
    from paper_2312_00407_b200.optim import zero_plan

    ps, offs = (C.c_size_t * N)(), (C.c_size_t * (N + 1))()
    O.ref_check(O.ref.ref_zero_plan(P, N, 2, ps, offs))
    ops, ooffs = (C.c_uint64 * N)(), (C.c_uint64 * (N + 1))()
    assert O.orc.orc_zero_plan(P, N, ops, ooffs) == 0
    mine = zero_plan(P, N, 2)
    assert list(ps) == list(ops) == mine[0]
    assert list(offs) == list(ooffs) == mine[1]
    if (P, N) == (10, 4):
        assert mine[0] == [3, 3, 2, 2]


# ---- the reference's own known-answer tests (test_optim.cpp) -----------------------------

def run_both(kind, n, p0, gseq, step_lr, **kw):
    cfg = cfg_for(kind, **kw)
    outs = []
    for mk in ([lambda: O.RefFlat(cfg, n)] if O.ref else []) + [
            lambda: O.OracleFlat(cfg, n, np.float64)]:
        opt, p = mk(), np.array(p0, np.float64)
        for g in gseq:
            opt.step(p, np.array(g, np.float64), step_lr)
        outs.append(p)
    return outs


def test_kat_adamw():  # test_optim.cpp:94-107
    for p in run_both(Kind.ADAMW, 1, [1.0], [[1.0]], 0.1, lr=0.1):
        assert p[0] == pytest.approx(0.9, rel=1e-7)
    for p in run_both(Kind.ADAMW, 3, [1, -2, 3], [[0, 0, 0]] * 4, 0.1, lr=0.1):
        assert list(p) == [1, -2, 3]


def test_kat_lion():  # test_optim.cpp:158-181
    for p in run_both(Kind.LION, 1, [1.0], [[1.0]], 0.1, lr=0.1):
        assert p[0] == pytest.approx(0.9, rel=1e-12)
    for p in run_both(Kind.LION, 1, [2.0], [[0.0]], 0.1, lr=0.1):
        assert p[0] == 2.0  # sign(0) = 0
    cfg = cfg_for(Kind.LION, lr=0.1)
    o, p = O.OracleFlat(cfg, 1), np.zeros(1)
    rng = np.random.default_rng(5)
    for _ in range(20):
        before = p[0]
        o.step(p, np.array([rng.normal(0, 100.0)]), 0.1)
        assert abs(p[0] - before) <= 0.1 + 1e-15


def test_kat_adan_first_step():  # test_optim.cpp:183-198
    expect = 1.0 - 0.05 * 0.7 / (math.sqrt(0.7 * 0.7) + 1e-8)
    for p in run_both(Kind.ADAN, 1, [1.0], [[0.7]], 0.05, lr=0.05):
        assert p[0] == pytest.approx(expect, rel=1e-12)
    if O.ref:
        assert O.RefFlat(cfg_for(Kind.ADAN), 10).state_bytes() == 4 * 10 * 8
        assert O.RefFlat(cfg_for(Kind.ADAMW), 10).state_bytes() == 2 * 10 * 8


def test_kat_sophia():  # test_optim.cpp:201-218
    for p in run_both(Kind.SOPHIA, 2, [1.0, -1.0], [[0.0, 0.0]], 0.02, lr=0.02):
        assert list(p) == [1.0, -1.0]
    cfg = cfg_for(Kind.SOPHIA, lr=0.02)
    o, p = O.OracleFlat(cfg, 1), np.array([0.3])
    rng = np.random.default_rng(11)
    for _ in range(30):
        before = p[0]
        o.step(p, np.array([rng.normal(0, 10.0)]), 0.02)
        assert abs(p[0] - before) <= 0.02 + 1e-15


def test_kat_scalar_references_100_steps():
    """test_optim.cpp:110-156: 100 N(0,1) steps, wd 0.01, theta0 0.5, vs independent
    scalar restatements of each update rule (RefAdamW .. RefSophia, :17-71)."""
    rng = np.random.default_rng(2024)
    gs = rng.normal(0, 1.0, 100)

    def ref_scalar(kind, c):
        th, m, v, n, h, gp = 0.5, 0.0, 0.0, 0.0, 0.0, 0.0
        out = []
        for t, g in enumerate(gs, start=1):
            if kind == Kind.ADAMW:
                m = c.beta1 * m + (1 - c.beta1) * g
                v = c.beta2 * v + (1 - c.beta2) * g * g
                mh, vh = m / (1 - c.beta1 ** t), v / (1 - c.beta2 ** t)
                th = th - c.lr * (mh / (math.sqrt(vh) + c.eps) + 0.01 * th)
            elif kind == Kind.LION:
                u = c.beta1 * m + (1 - c.beta1) * g
                s = 1.0 if u > 0 else (-1.0 if u < 0 else 0.0)
                th = th - c.lr * (s + 0.01 * th)
                m = c.beta2 * m + (1 - c.beta2) * g
            elif kind == Kind.ADAN:
                gd = 0.0 if t == 1 else g - gp
                m = c.beta1 * m + (1 - c.beta1) * g
                v = c.beta2 * v + (1 - c.beta2) * gd
                nu = g + c.beta2 * gd
                n = c.beta3 * n + (1 - c.beta3) * nu * nu
                mh, vh, nh = (m / (1 - c.beta1 ** t), v / (1 - c.beta2 ** t),
                              n / (1 - c.beta3 ** t))
                gp = g
                th = (th - c.lr * (mh + c.beta2 * vh) / (math.sqrt(nh) + c.eps)) / (
                    1 + c.lr * 0.01)
            else:
                m = c.beta1 * m + (1 - c.beta1) * g
                if (t - 1) % c.update_interval == 0:
                    h = c.beta2 * h + (1 - c.beta2) * g * g
                u = min(max(m / max(c.sophia_rho * h, c.eps), -1.0), 1.0)
                th = th - c.lr * u - c.lr * 0.01 * th
            out.append(th)
        return out

    for kind in FLAT_KINDS:
        c = cfg_for(kind, weight_decay=0.01)
        want = ref_scalar(kind, c)
        o, p = O.OracleFlat(c, 1), np.array([0.5])
        for g, w in zip(gs, want):
            o.step(p, np.array([g]), c.lr)
            assert abs(p[0] - w) < 1e-12


@needs_ref
def test_kat_adalomo_rank1_exact():  # test_optim.cpp:318-352
    av, bv = np.array([0.5, -1.5, 2.0]), np.array([1.0, 0.25, -2.0, 0.5])
    g = np.outer(av, bv).ravel()
    cfg = cfg_for(Kind.ADALOMO)
    for mk in (lambda: O.RefAdaLomo(cfg, [(3, 4)]), lambda: O.OracleAdaLomo(cfg, [(3, 4)])):
        st, p = mk(), np.ones(12)
        st.apply(0, p, g.copy(), 0.01)
        delta = 1.0 - p
        ratio = delta / (g / np.sqrt(g * g + cfg.eps))
        assert np.all(ratio > 0)
        np.testing.assert_allclose(ratio, ratio[0], rtol=1e-9)


def test_kat_state_bytes_and_validation():  # test_optim.cpp:354-388
    from paper_2312_00407_b200.optim import (ConfigError, PrecisionPolicy, parse_kind,
                                             state_bytes)

    fp16 = PrecisionPolicy()
    assert state_bytes(Kind.LOMO, 1000, fp16) == 0
    assert state_bytes(Kind.ADAMW, 100, fp16) == 1200
    assert state_bytes(Kind.ADAN, 100, fp16) - state_bytes(Kind.ADAMW, 100, fp16) == 400
    assert state_bytes(Kind.SOPHIA, 100, fp16) == state_bytes(Kind.ADAMW, 100, fp16)
    assert state_bytes(Kind.LION, 100, fp16) + 400 == state_bytes(Kind.ADAMW, 100, fp16)
    assert state_bytes(Kind.ADAMW, 100, PrecisionPolicy(4)) == 800
    assert state_bytes(Kind.ADALOMO, 8 * 16 + 32, fp16, [(8, 16), (32,)]) == (8 + 16) * 4 + 128
    with pytest.raises(ConfigError):
        state_bytes(Kind.ADALOMO, 10, fp16)
    cfg = cfg_for(Kind.ADAMW, lr=0.0)
    with pytest.raises(ConfigError):
        cfg.validate()
    cfg = cfg_for(Kind.ADAMW, beta1=1.0)
    with pytest.raises(ConfigError):
        cfg.validate()
    with pytest.raises(ConfigError, match="unknown optimizer kind 'sgd'"):
        parse_kind("sgd")
    assert parse_kind("adalomo") == Kind.ADALOMO


@needs_ref
def test_host_logic_matches_reference():
    """defaults_for / validate / state_bytes / kind names: product host code == reference."""
    from paper_2312_00407_b200 import optim

    for k in range(6):
        rc = O.Config()
        O.ref_check(O.ref.ref_defaults_for(k, C.byref(rc)))
        mine = O.Config.of(optim.OptimizerConfig.defaults_for(k))
        assert bytes(rc) == bytes(mine)
        assert O.ref.ref_kind_name(k).decode() == optim.kind_name(k)
        assert bool(O.ref.ref_is_fused(k)) == optim.is_fused(k)
    bad = [dict(lr=-1), dict(eps=0), dict(beta2=1.0), dict(beta3=-0.1), dict(weight_decay=-1),
           dict(update_interval=0)]
    for b in bad:
        c = cfg_for(Kind.ADAMW, **b)
        st = O.ref.ref_validate(C.byref(O.Config.of(c)))
        with pytest.raises(optim.ConfigError) as e:
            c.validate()
        assert st == 2 and O.ref.ref_last_error().decode() == str(e.value)
    shapes = [(8, 16), (32,), (5, 5, 2)]
    nd = (C.c_int * 3)(*[len(s) for s in shapes])
    dims = (C.c_int64 * 7)(*[d for s in shapes for d in s])
    for k in range(6):
        for pb, mc in [(2, 1), (4, 1), (2, 0)]:
            out = C.c_uint64()
            O.ref_check(O.ref.ref_state_bytes(k, 210, pb, 4, mc, 3, nd, dims, C.byref(out)))
            assert out.value == optim.state_bytes(k, 210, optim.PrecisionPolicy(pb, 4, bool(mc)),
                                                  shapes)


# ---- f32 restatement vs the f64 reference: the fp32 tolerance claim (tests/parity.py) ----


@needs_ref
@pytest.mark.parametrize("kind", FLAT_KINDS + ["sophia_m64"])
def test_f32_restatement_within_tolerance_of_reference(kind):
    """p, Δp and every state buffer within 1e-5 of the fp64 reference per element
    (tests/parity.py floors).  Sophia: the precise-m restatement (fp64 m); its fp32-m
    path is the separate, documented claim below."""
    import parity

    if kind == Kind.SOPHIA:
        pytest.skip("fp32-m Sophia: test_sophia_fp32_m_exceedance_is_bounded")
    n, steps, lr = 1 << 14, 20, 1e-3
    m64 = kind == "sophia_m64"
    cfg = cfg_for(Kind.SOPHIA if m64 else kind, weight_decay=0.01)
    p64 = O.synth(n, 2024, 0, 1, 0, 0, -6, 0, False, np.float64)
    p0, p32 = p64.copy(), p64.astype(np.float32)
    r = O.RefFlat(cfg, n)
    o = O.OracleSophiaM64(cfg, n) if m64 else O.OracleFlat(cfg, n, np.float32)
    for t in range(1, steps + 1):
        g32 = O.synth(n, 2024, 1, 1, t, 0, -7, 10, False, np.float32)
        r.step(p64, g32.astype(np.float64), lr)
        o.step(p32, g32, lr)
    parity.assert_flat_within(p32, p64, p0, lr, steps, o.state, r.buffers(), str(kind))


@needs_ref
def test_sophia_fp32_m_exceedance_is_bounded():
    """Sophia with fp32 m (the default product path): clamp(m / max(rho h, eps))
    amplifies m's fp32 cancellation error by 1/(rho h) in the unclamped band, so a few
    elements exceed the per-element bar -- measured 0.06 % of them, by <= 0.016 lr.  The
    claim for this path is that bound; precise-m (state "f32m64") meets the bar."""
    import parity

    n, steps, lr = 1 << 16, 20, 1e-3
    cfg = cfg_for(Kind.SOPHIA, weight_decay=0.01)
    p64 = O.synth(n, 2024, 0, 1, 0, 0, -6, 0, False, np.float64)
    p0, p32 = p64.copy(), p64.astype(np.float32)
    r, o = O.RefFlat(cfg, n), O.OracleFlat(cfg, n, np.float32)
    for t in range(1, steps + 1):
        g32 = O.synth(n, 2024, 1, 1, t, 0, -7, 10, False, np.float32)
        r.step(p64, g32.astype(np.float64), lr)
        o.step(p32, g32, lr)
    ex = parity.exceedance(p32, p64, p0, lr)
    assert 0 < ex["fraction"] <= 1e-3 and ex["max_abs_over_lr"] <= 0.02, ex
    # the state itself is within the bar: the drift is m / (rho h) amplification only
    e = parity.flat_errors(p32, p64, p0, lr, steps, o.state, r.buffers())
    assert e["m"] <= parity.TOL and e["h"] <= parity.TOL, e


def test_synth_generator_exact_grid():
    x = O.synth(1 << 16, 1, 1, 2, 3, 128, -7, 10, True)
    assert np.all(np.isfinite(x))
    frac0 = np.mean(x == 0)
    assert 0.0003 < frac0 < 0.002  # 2^-10 forced zeros (+ grid zeros)
    b = O.synth(4096, 1, 1, 2, 3, 0, -7, 10, False, "bf16")
    f = O.bf16_to_f32(b)
    assert np.array_equal(O.f32_to_bf16(f), b)  # bf16 grid values are exact
