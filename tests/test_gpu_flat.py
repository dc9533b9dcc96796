"""GPU parity of the stored-state optimizers (AdamW / Lion / Adan / Sophia) through
the C-ABI against the oracle: bit-exact vs the fp32 restatement, bit-exact vs the
compiled reference in f64 mode, fp32-tolerance vs the reference."""
import numpy as np
import pytest

import oracle as O
from paper_2312_00407_b200 import optim
from paper_2312_00407_b200.optim import Kind, OptimizerConfig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FLAT = [Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA]


def cfg_for(kind, **kw):
    c = OptimizerConfig.defaults_for(kind)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("kind", FLAT)
@pytest.mark.parametrize("n", [1, 13, 4096 + 5, 1 << 20])
def test_f32_bit_exact_vs_restatement(kind, n):
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=3)
    p = O.synth(n, 2024, 0, 1, 0, 0, -6, 0, False)
    gpu_p = dev(p)
    opt = optim.FlatOptimizer(cfg, n)
    orc = O.OracleFlat(cfg, n, np.float32)
    for t in range(1, 8):
        g = O.synth(n, 2024, 1, 1, t, 0, -7, 10, False)
        opt.step(gpu_p, dev(g), 1e-3)
        orc.step(p, g, 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(gpu_p.cpu().numpy(), p)
    bufs = opt.buffers()
    assert [b[0] for b in bufs] == list(orc.state)
    for name, t in bufs:
        assert bits_equal(t.cpu().numpy(), orc.state[name]), name
    assert opt.steps_taken() == 7


@pytest.mark.parametrize("kind", FLAT)
def test_unaligned_views_bit_exact(kind):
    """ZeRO shard edges: params / grads at odd element offsets (the state takes their
    alignment phase at the first step; a short head is peeled, the rest vectorised)."""
    n, off = 10007, 3
    cfg = cfg_for(kind, weight_decay=0.01)
    pbig = O.synth(n + off, 7, 0, 2, 0, 0, -6, 0, False)
    gbig = O.synth(n + off, 7, 1, 2, 1, 0, -7, 10, False)
    tp, tg = dev(pbig), dev(gbig)
    opt = optim.FlatOptimizer(cfg, n)
    opt.step(tp[off:], tg[off:], 1e-3)
    orc = O.OracleFlat(cfg, n, np.float32)
    p = pbig[off:].copy()
    orc.step(p, gbig[off:].copy(), 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp[off:].cpu().numpy(), p)
    assert bits_equal(tp[:off].cpu().numpy(), pbig[:off])  # untouched


@pytest.mark.parametrize("kind", FLAT)
def test_bf16_grads_and_mixed_param_out(kind):
    n = 70001
    cfg = cfg_for(kind, weight_decay=0.01)
    p = O.synth(n, 3, 0, 0, 0, 0, -6, 0, False)
    gb = O.synth(n, 3, 1, 0, 1, 0, -7, 10, False, "bf16")
    tp, tpo = dev(p), torch.empty(n, dtype=torch.bfloat16, device="cuda")
    tg = dev(gb).view(torch.bfloat16)
    opt = optim.FlatOptimizer(cfg, n)
    opt.step_mixed(tp, tg, tpo, 1e-3)
    orc = O.OracleFlat(cfg, n, np.float32)
    orc.step(p, O.bf16_to_f32(gb), 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)
    assert bits_equal(tpo.view(torch.int16).cpu().numpy().view(np.uint16), O.f32_to_bf16(p))


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("kind", FLAT)
def test_f64_mode_bit_exact_vs_compiled_reference(kind):
    """state_dtype f64: every element identical to minicollie::optim::FlatOptimizer."""
    n = 50000 + 3
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=4)
    p = O.synth(n, 11, 0, 0, 0, 0, -6, 0, False, np.float64)
    tp = dev(p)
    opt = optim.FlatOptimizer(cfg, n, state_dtype="f64")
    r = O.RefFlat(cfg, n)
    for t in range(1, 13):
        g = O.synth(n, 11, 1, 0, t, 0, -7, 10, False, np.float64)
        opt.step(tp, dev(g), 1e-3)
        r.step(p, g, 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)
    rb = r.buffers()
    for name, t in opt.buffers():
        assert bits_equal(t.cpu().numpy(), rb[name]), name


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("kind", list(FLAT) + ["sophia_m64"])
def test_f32_within_tolerance_of_reference(kind):
    """The product path vs the fp64 reference after 20 steps: p, Δp and every state
    buffer within 1e-5 per element (tests/parity.py floors).  Sophia's fp32-m path is
    held to its documented exceedance bound; its precise-m state ("f32m64") meets the
    per-element bar and is bit-exact to its restatement."""
    import parity

    n, lr, steps = 1 << 16, 1e-3, 20
    m64 = kind == "sophia_m64"
    cfg = cfg_for(Kind.SOPHIA if m64 else kind, weight_decay=0.01)
    p64 = O.synth(n, 2024, 0, 1, 0, 0, -6, 0, False, np.float64)
    p0 = p64.copy()
    p32 = p64.astype(np.float32)
    tp = dev(p32)
    opt = optim.FlatOptimizer(cfg, n, state_dtype="f32m64" if m64 else "f32")
    r = O.RefFlat(cfg, n)
    o = O.OracleSophiaM64(cfg, n) if m64 else None
    for t in range(1, steps + 1):
        g = O.synth(n, 2024, 1, 1, t, 0, -7, 10, False)
        opt.step(tp, dev(g), lr)
        r.step(p64, g.astype(np.float64), lr)
        if o is not None:
            o.step(p32, g, lr)
    torch.cuda.synchronize()
    got = tp.cpu().numpy()
    state = {nm: t.cpu().numpy() for nm, t in opt.buffers()}
    if m64:
        assert bits_equal(got, p32)
        assert bits_equal(state["m"], o.state["m"]) and bits_equal(state["h"], o.state["h"])
        assert state["m"].dtype == np.float64
    name = "sophia_m64" if m64 else Kind(kind).name.lower()
    ex = parity.exceedance(got, p64, p0, lr)
    ex.update(parity.flat_errors(got, p64, p0, lr, steps, state, r.buffers()))
    ex["case"] = f"{n} elements, {steps} steps, lr {lr}, wd 0.01, vs the fp64 reference"
    parity.record(name, ex)
    if kind == Kind.SOPHIA:
        assert ex["fraction"] <= 1e-3 and ex["max_abs_over_lr"] <= 0.02, ex
        return
    parity.assert_flat_within(got, p64, p0, lr, steps, state, r.buffers(), str(kind))


@pytest.mark.parametrize("kind", FLAT)
def test_host_span_path_equals_device_path(kind):
    """The reference's std::span overload (mco_flat_step_host) == device step."""
    n = (1 << 24) + 12345  # > one pipeline chunk
    cfg = cfg_for(kind, weight_decay=0.01)
    p = O.synth(n, 5, 0, 0, 0, 0, -6, 0, False)
    g = O.synth(n, 5, 1, 0, 1, 0, -7, 10, False)
    a, b = optim.FlatOptimizer(cfg, n), optim.FlatOptimizer(cfg, n)
    hp = p.copy()
    a.step(hp, g, 1e-3)
    tp = dev(p)
    b.step(tp, dev(g), 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(hp, tp.cpu().numpy())


def test_contract_errors_match_reference_messages():
    cfg = cfg_for(Kind.ADAMW)
    opt = optim.FlatOptimizer(cfg, 8)
    p = torch.zeros(8, device="cuda")
    with pytest.raises(optim.ContractError,
                       match="optimizer step: params/grads length mismatch: 8 vs 7"):
        opt.step(p, torch.zeros(7, device="cuda"), 0.1)
    assert opt.steps_taken() == 0  # optim.cpp:101-104: checked before ++t
    with pytest.raises(optim.ContractError):
        opt.step(torch.zeros(9, device="cuda"), torch.zeros(9, device="cuda"), 0.1)
    with pytest.raises(optim.ContractError):
        opt.step(p.double(), p.double(), 0.1)  # f64 data into an f32 optimizer


def test_kat_through_gpu():
    """test_optim.cpp known answers through the GPU path (f32 and f64 modes)."""
    for sd, dt in (("f32", torch.float32), ("f64", torch.float64)):
        c = cfg_for(Kind.ADAMW, lr=0.1)
        o = optim.FlatOptimizer(c, 1, state_dtype=sd)
        p = torch.ones(1, dtype=dt, device="cuda")
        o.step(p, torch.ones(1, dtype=dt, device="cuda"), 0.1)
        assert p.item() == pytest.approx(0.9, rel=1e-7)
        c = cfg_for(Kind.LION, lr=0.1)
        o = optim.FlatOptimizer(c, 1, state_dtype=sd)
        p = torch.full((1,), 2.0, dtype=dt, device="cuda")
        o.step(p, torch.zeros(1, dtype=dt, device="cuda"), 0.1)
        assert p.item() == 2.0
        c = cfg_for(Kind.SOPHIA, lr=0.02)
        o = optim.FlatOptimizer(c, 2, state_dtype=sd)
        p = torch.tensor([1.0, -1.0], dtype=dt, device="cuda")
        o.step(p, torch.zeros(2, dtype=dt, device="cuda"), 0.02)
        assert p.tolist() == [1.0, -1.0]
    c = cfg_for(Kind.ADAN)
    assert optim.FlatOptimizer(c, 10, state_dtype="f64").state_bytes_runtime() == 4 * 10 * 8
    assert optim.FlatOptimizer(c, 10).state_bytes_runtime() == 4 * 10 * 4


def test_sampled_parity_at_scale():
    """A 2^30-element AdamW step (4 GiB per buffer), checked on sampled slices that
    the oracle regenerates from the counter-based generator."""
    n = 1 << 30
    cfg = cfg_for(Kind.ADAMW, weight_decay=0.01)
    tp = torch.empty(n, device="cuda")
    tg = torch.empty(n, device="cuda")
    optim.synth_fill(tp, 2024, 0, 9, 0, 0, -6)
    opt = optim.FlatOptimizer(cfg, n)
    for t in (1, 2):
        optim.synth_fill(tg, 2024, 1, 9, t, 0, -7, 10)
        opt.step(tp, tg, 1e-3)
    torch.cuda.synchronize()
    key_p, G = O.orc.orc_synth_key(2024, 0, 9, 0), 0x9E3779B97F4A7C15
    for start in (0, 123456789, n - 4096):
        m = 4096
        p = np.empty(m, np.float32)
        O.orc.orc_synth_f32(O._ptr(p), m, (key_p + start * G) % (1 << 64), 0, -6, 0, 0)
        orc = O.OracleFlat(cfg, m, np.float32)
        for t in (1, 2):
            g = np.empty(m, np.float32)
            key_g = O.orc.orc_synth_key(2024, 1, 9, t)
            O.orc.orc_synth_f32(O._ptr(g), m, (key_g + start * G) % (1 << 64), 0, -7, 10, 0)
            orc.step(p, g, 1e-3)
        assert bits_equal(tp[start:start + m].cpu().numpy(), p)
    del tp, tg
    torch.cuda.empty_cache()


def test_state_bytes_match_device_memory():
    """f3: state_bytes_runtime equals the device memory the optimizer allocates."""
    n = 1 << 26
    for kind, nbuf in ((Kind.ADAMW, 2), (Kind.LION, 1), (Kind.ADAN, 4), (Kind.SOPHIA, 2)):
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        opt = optim.FlatOptimizer(cfg_for(kind), n)
        torch.cuda.synchronize()
        used = free0 - torch.cuda.mem_get_info()[0]
        assert opt.state_bytes_runtime() == nbuf * n * 4
        assert abs(used - opt.state_bytes_runtime()) <= (4 << 20) * nbuf  # allocation granularity
        del opt


def test_empty_step_advances_counter_like_the_reference():
    # optim.cpp:100-112: empty spans pass the length check, ++t, no element loop
    opt = optim.FlatOptimizer(cfg_for(Kind.ADAN), 0)
    e = torch.empty(0, device="cuda")
    opt.step(e, e, 1e-3)
    assert opt.steps_taken() == 1
    optim.lomo_apply(e, e, 1e-3)
    assert optim.sumsq(e).item() == 0.0


@pytest.fixture
def flat_variant():
    """Switch the stored-state kernels' data-movement variant for one test."""
    prev = optim.flat_variant()
    yield optim.set_flat_variant
    optim.set_flat_variant(prev)


@pytest.mark.parametrize("variant", ["ldg", "tma", "tma_s3", "tma24", "tma8", "tma_e2", "tma_hint", "tma_ds", "pf", "w4m4", "l2pf2"])
@pytest.mark.parametrize("kind", FLAT)
@pytest.mark.parametrize("n", [2048, 3 * 3072 + 77, (1 << 20) + 5])
def test_kernel_variants_bit_exact(flat_variant, variant, kind, n):
    """Every data-movement variant (TMA bulk-copy pipeline included) produces the
    restatement's bits: tail elements, Adan's t == 1, Sophia refresh / non-refresh,
    mixed bf16 replica output."""
    flat_variant(variant)
    assert optim.flat_variant() == variant
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=3)
    p = O.synth(n, 77, 0, 3, 0, 0, -6, 0, False)
    tp, tpo = dev(p), torch.empty(n, dtype=torch.bfloat16, device="cuda")
    opt = optim.FlatOptimizer(cfg, n)
    orc = O.OracleFlat(cfg, n, np.float32)
    for t in range(1, 6):
        g = O.synth(n, 77, 1, 3, t, 0, -7, 10, False)
        if t == 5:
            opt.step_mixed(tp, dev(g), tpo, 1e-3)
        else:
            opt.step(tp, dev(g), 1e-3)
        orc.step(p, g, 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)
    assert bits_equal(tpo.view(torch.int16).cpu().numpy().view(np.uint16), O.f32_to_bf16(p))
    for name, t in opt.buffers():
        assert bits_equal(t.cpu().numpy(), orc.state[name]), name



@pytest.mark.parametrize("variant", ["tma", "ldg"])
@pytest.mark.parametrize("kind", FLAT)
@pytest.mark.parametrize("g_log2", [-66, -100, -130])
def test_tiny_gradients_bit_exact(flat_variant, variant, kind, g_log2):
    """Gradients of 2^-66 .. 2^-130 (squares and EMAs subnormal, g itself subnormal at
    the end): the subnormal-safe sqrt(x/c) + eps keeps the restatement's bits while
    avoiding the IEEE slow paths."""
    flat_variant(variant)
    n = (1 << 20) + 5
    cfg = cfg_for(kind, weight_decay=0.01)
    p = O.synth(n, 31, 0, 4, 0, 0, -6, 0, False)
    tp = dev(p)
    opt = optim.FlatOptimizer(cfg, n)
    orc = O.OracleFlat(cfg, n, np.float32)
    for t in range(1, 4):
        g = O.synth(n, 31, 1, 4, t, 0, g_log2, 10, False)
        opt.step(tp, dev(g), 1e-3)
        orc.step(p, g, 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)
    for name, t in opt.buffers():
        assert bits_equal(t.cpu().numpy(), orc.state[name]), name


@pytest.mark.parametrize("variant", ["tma", "ldg"])
@pytest.mark.parametrize("kind", FLAT)
def test_phase_peeling_cases_bit_exact(flat_variant, variant, kind):
    """Views at every phase 1..7, mismatched param / grad phases (scalar path), state
    handed out before the first step (layout frozen), the mixed step with a bf16 replica
    at an odd offset, and LOMO on views: all give the restatement's bits."""
    flat_variant(variant)
    n = 3 * 4096 + 11
    cfg = cfg_for(kind, weight_decay=0.01)
    P = O.synth(n + 16, 8, 0, 5, 0, 0, -6, 0, False)
    G = O.synth(n + 16, 8, 1, 5, 1, 0, -7, 10, False)
    tP, tG = dev(P), dev(G)
    for po, go, expose in [(ph, ph, False) for ph in range(1, 8)] + [(3, 5, False), (2, 2, True)]:
        p = P[po:po + n].copy()
        tp = tP.clone()[po:po + n]
        opt = optim.FlatOptimizer(cfg, n)
        if expose:
            _ = opt.buffers()
        orc = O.OracleFlat(cfg, n, np.float32)
        for t in (1, 2):
            opt.step(tp, tG[go:go + n], 1e-3)
            orc.step(p, G[go:go + n].copy(), 1e-3)
        torch.cuda.synchronize()
        assert bits_equal(tp.cpu().numpy(), p), (po, go, expose)
        for name, buf in opt.buffers():
            assert bits_equal(buf.cpu().numpy(), orc.state[name]), (po, go, name)
    # mixed step: fp32 master (aligned) + bf16 replica slice at offset 3: phases differ
    master = O.synth(n, 9, 0, 5, 0, 0, -6, 0, False)
    tm = dev(master)
    rep = torch.empty(n + 8, dtype=torch.bfloat16, device="cuda")[3:3 + n]
    opt = optim.FlatOptimizer(cfg, n)
    orc = O.OracleFlat(cfg, n, np.float32)
    opt.step_mixed(tm, tG[:n], rep, 1e-3)
    orc.step(master, G[:n].copy(), 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tm.cpu().numpy(), master)
    assert bits_equal(rep.view(torch.int16).cpu().numpy().view(np.uint16), O.f32_to_bf16(master))


@pytest.mark.parametrize("off", [1, 5])
def test_lomo_views_bit_exact(off):
    n = 50000
    P = O.synth(n + 8, 4, 0, 0, 0, 0, -6, 0, False)
    G = O.synth(n + 8, 4, 1, 0, 1, 0, -7, 10, False)
    tp = dev(P)[off:off + n]
    optim.lomo_apply(tp, dev(G)[off:off + n], 1e-2, 0.5)
    p = P[off:off + n].copy()
    O.orc.orc_lomo_f32(O._ptr(p), O._ptr(G[off:off + n].copy()), n, 1e-2, 0.5)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)


@pytest.mark.parametrize("variant", ["tma", "ldg"])
@pytest.mark.parametrize("kind", FLAT)
def test_bf16_grads_both_paths_bit_exact(flat_variant, variant, kind):
    """bf16 gradients with fp32 state on the TMA pipeline (bf16 gradient tiles) and on
    the LDG kernel, plain and mixed (bf16 replica out), tail included."""
    flat_variant(variant)
    n = 5 * 2048 + 37
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=2)
    p = O.synth(n, 13, 0, 6, 0, 0, -6, 0, False)
    tp, tpo = dev(p), torch.empty(n, dtype=torch.bfloat16, device="cuda")
    opt = optim.FlatOptimizer(cfg, n)
    orc = O.OracleFlat(cfg, n, np.float32)
    for t in range(1, 5):
        gb = O.synth(n, 13, 1, 6, t, 0, -7, 10, False, "bf16")
        tg = dev(gb).view(torch.bfloat16)
        if t % 2:
            opt.step(tp, tg, 1e-3)
        else:
            opt.step_mixed(tp, tg, tpo, 1e-3)
        orc.step(p, O.bf16_to_f32(gb), 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)
    assert bits_equal(tpo.view(torch.int16).cpu().numpy().view(np.uint16), O.f32_to_bf16(p))
    for name, t in opt.buffers():
        assert bits_equal(t.cpu().numpy(), orc.state[name]), name


@pytest.mark.parametrize("gdt", ["f32", "bf16"])
@pytest.mark.parametrize("kind", FLAT)
@pytest.mark.parametrize("n", [4 * 2048, 5 * 2048 + 13])
def test_gradient_phase_shift_bit_exact(kind, gdt, n):
    """A gradient at another alignment phase than the parameters (every pair of phases
    0..7; fp32 and bf16 gradients): the TMA pipeline reads the gradient shifted
    (flat_tma_kernel gsh) instead of falling back to the scalar path -- same bits as the
    restatement, including n a whole number of tiles (the shifted last tile joins the
    scalar tail)."""
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=2)
    P = O.synth(n + 16, 12, 0, 6, 0, 0, -6, 0, False)
    G = [O.synth(n + 16, 12, 1, 6, t, 0, -7, 10, False) for t in (1, 2, 3)]
    if gdt == "bf16":  # bf16-valued: the restatement reads the same gradients as floats
        G = [O.bf16_to_f32(O.f32_to_bf16(x)) for x in G]
    tG = [dev(x) if gdt == "f32" else dev(x).to(torch.bfloat16) for x in G]
    for po in range(8):
        for go in range(8):
            if po == go:
                continue
            p = P[po:po + n].copy()
            tp = dev(P)[po:po + n]
            opt = optim.FlatOptimizer(cfg, n)
            orc = O.OracleFlat(cfg, n, np.float32)
            for t in range(3):
                opt.step(tp, tG[t][go:go + n], 1e-3)
                orc.step(p, G[t][go:go + n].copy(), 1e-3)
            torch.cuda.synchronize()
            assert bits_equal(tp.cpu().numpy(), p), (po, go)
            for name, buf in opt.buffers():
                assert bits_equal(buf.cpu().numpy(), orc.state[name]), (po, go, name)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_lomo_gradient_phase_shift_bit_exact(dt):
    """LOMO with the gradient at another phase than the parameters (lomo_tma_kernel
    gsh), every pair of phases: the restatement's bits."""
    n = 3 * 4096 + 8  # whole tiles (+8: the shifted last tile fits for some phases only)
    sd = np.float32 if dt == "f32" else "bf16"
    P = O.synth(n + 16, 13, 0, 0, 0, 0, -6, 0, False, sd)
    G = O.synth(n + 16, 13, 1, 0, 1, 0, -7, 10, False, sd)
    orc = O.orc.orc_lomo_f32 if dt == "f32" else O.orc.orc_lomo_bf16
    for po in range(8):
        for go in range(8):
            if po == go:
                continue
            tp = dev(P) if dt == "f32" else dev(P).view(torch.bfloat16)
            tg = dev(G) if dt == "f32" else dev(G).view(torch.bfloat16)
            optim.lomo_apply(tp[po:po + n], tg[go:go + n], 1e-2, 0.5)
            p = P[po:po + n].copy()
            orc(O._ptr(p), O._ptr(G[go:go + n].copy()), n, 1e-2, 0.5)
            torch.cuda.synchronize()
            got = tp[po:po + n].cpu().numpy() if dt == "f32" else \
                tp[po:po + n].view(torch.int16).cpu().numpy()
            assert bits_equal(got, p), (po, go)


@pytest.mark.parametrize("kind", FLAT)
def test_params_and_state_at_different_phases_bit_exact(kind):
    """State laid out before the first step (buffers() handed out: its phase is frozen at
    the allocation's) against parameters / gradients at other phases: the step runs as a
    one-tensor list step on the TMA list pipeline (every stream read and written at its
    own phase) -- the restatement's bits, state included."""
    n = 5 * 2048 + 13
    cfg = cfg_for(kind, weight_decay=0.01, update_interval=2)
    P = O.synth(n + 16, 21, 0, 7, 0, 0, -6, 0, False)
    G = [O.synth(n + 16, 21, 1, 7, t, 0, -7, 10, False) for t in (1, 2, 3)]
    for po, go in [(3, 3), (1, 6), (5, 0), (0, 7)]:
        p = P[po:po + n].copy()
        tp = dev(P)[po:po + n]
        tG = [dev(x) for x in G]
        opt = optim.FlatOptimizer(cfg, n)
        _ = opt.buffers()  # layout frozen at phase 0
        orc = O.OracleFlat(cfg, n, np.float32)
        for t in range(3):
            opt.step(tp, tG[t][go:go + n], 1e-3)
            orc.step(p, G[t][go:go + n].copy(), 1e-3)
        torch.cuda.synchronize()
        assert bits_equal(tp.cpu().numpy(), p), (po, go)
        for name, buf in opt.buffers():
            assert bits_equal(buf.cpu().numpy(), orc.state[name]), (po, go, name)


@pytest.mark.parametrize("gdt", ["f32", "bf16"])
@pytest.mark.parametrize("n,off", [(2048, 0), (5 * 2048 + 77, 0), (3 * 2048 + 5, 3), (1000, 0)])
def test_sophia_precise_m_paths_bit_exact(gdt, n, off):
    """Sophia precise-m (fp64 m) on the bulk-copy pipeline (aligned, whole tiles + tail)
    and on the LDG kernel (views off the 16 B grid, less than a tile): the restatement's
    bits for p, m and h over refresh and non-refresh steps, fp32 and bf16 gradients."""
    cfg = cfg_for(Kind.SOPHIA, weight_decay=0.01, update_interval=2)
    P = O.synth(n + 8, 31, 0, 2, 0, 0, -6, 0, False)
    p = P[off:off + n].copy()
    tp = dev(P)[off:off + n]
    opt = optim.FlatOptimizer(cfg, n, state_dtype="f32m64")
    orc = O.OracleSophiaM64(cfg, n)
    for t in range(1, 5):
        g = O.synth(n + 8, 31, 1, 2, t, 0, -7, 10, False)
        if gdt == "bf16":
            g = O.bf16_to_f32(O.f32_to_bf16(g))
        tg = dev(g) if gdt == "f32" else dev(g).to(torch.bfloat16)
        opt.step(tp, tg[off:off + n], 1e-3)
        orc.step(p, g[off:off + n].copy(), 1e-3)
    torch.cuda.synchronize()
    assert bits_equal(tp.cpu().numpy(), p)
    st = dict(opt.buffers())
    assert bits_equal(st["m"].cpu().numpy(), orc.state["m"])
    assert bits_equal(st["h"].cpu().numpy(), orc.state["h"])
