#!/usr/bin/env python3
"""Single-GPU measurements of BASELINE.json configs 3-5 (bench.py measures config 2).

  c3        AdaLomo, factored moments + global grad-norm clip, LLaMA-13B shapes (1 GPU)
  c4-shard  one rank's ZeRO shard at N=8 of the 65B set: Sophia, mixed precision
            (fp32 master/state/grads, bf16 parameter copy written for the all-gather);
            and Adan mixed on the 65B-L16 subset's N=8 shard (full 65B Adan state does
            not fit 180 GB per rank at N=8)
  c5-shard  one rank's shard at N=8 of the Llama-2-70B (GQA) set: LOMO with bf16
            params/grads and the global grad-norm clip (sum of squares + clipped update;
            the one-scalar all-reduce between them is not present on one GPU)

Each line: params/s for that launch, algorithmic bytes, achieved GB/s, fraction of the
measured HBM copy bandwidth.  Timed with CUDA events after warm-up; inputs > L2.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, warmup, steps):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def line(name, n, ms, bpp, extra=None):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    gbs = bpp * n / (ms * 1e-3) / 1e9
    d = {"config": name, "params": n, "ms": round(ms, 3), "params_per_s": n / (ms * 1e-3),
         "bytes_per_param": bpp, "achieved_gbs": round(gbs, 1), "hbm_peak_gbs": peak,
         "frac": round(gbs / peak, 4)}
    d.update(extra or {})
    print(json.dumps(d), flush=True)


def main():
    import gc

    import torch

    from paper_2312_00407_b200 import optim, registry
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    W, K = 2, 5
    which = sys.argv[1:] or ["c3", "c4", "c5", "hooks", "bf16", "cliff", "phases"]

    if "c3" in which:
        m = registry.LLAMA_13B
        shapes, n = m.shapes(), m.param_count()
        p = torch.empty(n, device="cuda")
        g = torch.empty(n, device="cuda")
        registry.fill_params(p, shapes)
        registry.fill_grads(g, shapes, 1)
        cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
        cfg.lr = 5e-4
        st = optim.AdaLomoState(cfg, shapes, grad_clip=1.0)
        ms = timed(lambda: st.apply_all(p, g, cfg.lr), W, K)
        line("c3 adalomo+clip llama-13b 1xB200", n, ms, 24,
             {"tensors": len(shapes), "state_floats": st.state_bytes_runtime() // 8})
        del st, p, g
        gc.collect()
        torch.cuda.empty_cache()

    if "c4" in which:
        for kind, model, bpp in ((Kind.SOPHIA, registry.LLAMA_65B, 26),
                                 (Kind.ADAN, registry.LLAMA_65B_L16, 46)):
            n = optim.zero_plan(model.param_count(), 8)[0][0]
            master = torch.empty(n, device="cuda")
            g = torch.empty(n, device="cuda")
            out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            optim.synth_fill(master, registry.SEED, 0, 1, 0, 0, -6)
            optim.synth_fill(g, registry.SEED, 1, 1, 1, 0, -7, 10)
            cfg = OptimizerConfig.defaults_for(kind)
            cfg.lr = 1e-4 if kind == Kind.SOPHIA else 5e-5
            opt = optim.FlatOptimizer(cfg, n)
            ms = timed(lambda: opt.step_mixed(master, g, out, cfg.lr), W, K)
            line(f"c4 {optim.kind_name(kind)} mixed, rank shard of {model.name} at N=8", n, ms,
                 bpp, {"note": "Sophia: refresh steps every 10 write h (+4 B/param)"
                       if kind == Kind.SOPHIA else "fp32 master/state/grads, bf16 out"})
            del opt, master, g, out
            gc.collect()
            torch.cuda.empty_cache()

    if "c5" in which:
        model = registry.LLAMA2_70B
        n = optim.zero_plan(model.param_count(), 8)[0][0]
        p = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        g = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        optim.synth_fill(p, registry.SEED, 0, 2, 0, 0, -6)
        optim.synth_fill(g, registry.SEED, 1, 2, 1, 0, -7, 10)
        ms = timed(lambda: optim.lomo_step(p, g, 1e-2, clip=1.0), W, K)
        line("c5 lomo bf16 + global clip, rank shard of llama2-70b at N=8", n, ms, 8,
             {"passes": "sum of squares (2 B/param) + clipped update (6 B/param)"})
        ms = timed(lambda: optim.lomo_apply(p, g, 1e-2, 1.0), W, K)
        line("c5 lomo bf16 no clip, rank shard of llama2-70b at N=8", n, ms, 6)
        del p, g
        gc.collect()
        torch.cuda.empty_cache()

    if "hooks" in which:
        hooks_7b(W, K)

    if "cliff" in which:
        cliff(W, K)

    if "phases" in which:
        phases(W, K)

    if "bf16" in which:  # AdaLomo on bf16 parameters and gradients (12 B/param)
        m = registry.LLAMA_7B
        shapes, n = m.shapes(), m.param_count()
        p = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        g = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        tmp = torch.empty(n // 4 + 1, device="cuda")
        off = 0  # fp32 synthetic values, rounded to bf16, a slice at a time
        for k, s_ in enumerate(shapes):
            cnt = int(torch.tensor(s_).prod())
            for a in range(0, cnt, tmp.numel()):
                b = min(cnt, a + tmp.numel())
                t = tmp[:b - a]
                if len(s_) == 2:
                    optim.synth_fill(t, registry.SEED, 0, k, 0, 0, -6)
                else:
                    t.fill_(1.0)
                p[off + a:off + b].copy_(t)
            off += cnt
        registry.fill_grads(g, shapes, 1)
        del tmp
        cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
        st = optim.AdaLomoState(cfg, shapes)
        ms = timed(lambda: st.apply_all(p, g, 5e-4), W, K)
        line("adalomo bf16 params + bf16 grads, llama-7b", n, ms, 12)


def phases(W, K):
    """Stored-state / LOMO steps whose gradient sits at another alignment phase than the
    parameters (a gradient view one element in): the TMA pipeline reads it shifted
    (round 1: the whole step took the scalar path)."""
    import torch

    from paper_2312_00407_b200 import optim
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    n = 1 << 30
    p = torch.empty(n, device="cuda")
    gb = torch.empty(n + 8, device="cuda")
    optim.synth_fill(p, 1, 0, 0, 0, 0, -6)
    optim.synth_fill(gb, 1, 1, 0, 1, 0, -7, 10)
    for kind, bpp in ((Kind.ADAMW, 28), (Kind.ADAN, 44)):
        cfg = OptimizerConfig.defaults_for(kind)
        opt = optim.FlatOptimizer(cfg, n)
        for go in (0, 1):
            g = gb[go:go + n]
            ms = timed(lambda: opt.step(p, g, 1e-5), W, K)
            line(f"{optim.kind_name(kind)} 2^30, gradient at element offset {go}", n, ms, bpp)
        del opt
    for go in (0, 1):
        g = gb[go:go + n]
        ms = timed(lambda: optim.lomo_apply(p, g, 1e-3, 1.0), W, K)
        line(f"lomo 2^30, gradient at element offset {go}", n, ms, 12)
    del p, gb
    # list form over separate tensors: a (7,) tensor first shifts every later tensor's
    # state off its parameters' 16 B phase (round 1: those tensors took the scalar path)
    for lead in (0, 7):
        shapes = ([(lead,)] if lead else []) + [(4096, 4096)] * 24
        ps = [torch.empty(s_, device="cuda").normal_(0, 0.02) for s_ in shapes]
        gs = [torch.empty(s_, device="cuda").normal_(0, 1e-3) for s_ in shapes]
        m = sum(x.numel() for x in ps)
        cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
        opt = optim.FlatOptimizer(cfg, m)
        ms = timed(lambda: opt.step_list(ps, gs, 1e-5), W, K)
        line(f"adamw list form, 24 x 4096^2 tensors{' after a (7,) tensor' if lead else ''}",
             m, ms, 28)
        del ps, gs, opt


def cliff(W, K):
    """AdaLomo's per-tensor vector path: a (7,) vector ahead of two 7B decoder layers
    shifts every later flat offset off the 8-element grid.  Before the per-tensor split
    the whole call ran scalar (6.3 vs 2.5 ms); now only the shifted tensors do."""
    import torch

    from paper_2312_00407_b200 import optim, registry
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    layer = registry.LLAMA_7B.shapes()[1:10]  # one decoder layer (9 tensors)
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    for name, shapes in (("aligned", layer + layer), ("(7,) first", [(7,)] + layer + layer),
                         ("(7,) mid", layer + [(7,)] + layer)):
        n = sum(int(torch.tensor(s_).prod()) for s_ in shapes)
        p = torch.empty(n, device="cuda")
        g = torch.empty(n, device="cuda")
        registry.fill_params(p, shapes)
        registry.fill_grads(g, shapes, 1)
        st = optim.AdaLomoState(cfg, shapes)
        ms = timed(lambda: st.apply_all(p, g, 5e-4), W, K)
        line(f"adalomo 2 llama-7b layers, {name}", n, ms, 24, {"tensors": len(shapes)})
        del st, p, g


def hooks_7b(W, K):
    """The per-tensor (backward-hook) forms of LOMO and AdaLomo over
    the 7B set, one call per tensor in reverse registry order as backward produces
    them, against the multi-tensor flat forms: the per-call overhead of the hook path."""
    import torch

    from paper_2312_00407_b200 import optim, registry
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    m = registry.LLAMA_7B
    shapes, n = m.shapes(), m.param_count()
    p = torch.empty(n, device="cuda")
    g = torch.empty(n, device="cuda")
    registry.fill_params(p, shapes)
    registry.fill_grads(g, shapes, 1)
    offs = [0]
    for s in shapes:
        offs.append(offs[-1] + int(torch.tensor(s).prod()))
    views = [(p[offs[k]:offs[k + 1]], g[offs[k]:offs[k + 1]]) for k in range(len(shapes))]
    order = list(reversed(range(len(shapes))))

    def lomo_hooks():
        for k in order:
            optim.lomo_apply(views[k][0], views[k][1], 1e-2, 1.0)

    ms = timed(lomo_hooks, W, K)
    line("hook-form lomo, llama-7b (291 calls)", n, ms, 12, {"calls": len(shapes)})
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    st = optim.AdaLomoState(cfg, shapes)

    def ada_hooks():
        for k in order:
            st.apply(k, views[k][0], views[k][1], 5e-4)

    ms = timed(ada_hooks, W, K)
    line("hook-form adalomo, llama-7b (291 calls)", n, ms, 24, {"calls": len(shapes)})
    bucket = 32  # the bucketed hook path: consecutive tensors in one list call

    def ada_buckets():
        for hi in range(len(shapes), 0, -bucket):
            lo = max(0, hi - bucket)
            st.apply_list(lo, [views[k][0] for k in range(lo, hi)],
                          [views[k][1] for k in range(lo, hi)], 5e-4)

    ms = timed(ada_buckets, W, K)
    line(f"hook-form adalomo, buckets of {bucket} tensors (list form), llama-7b", n, ms, 24,
         {"calls": (len(shapes) + bucket - 1) // bucket})
    ms = timed(lambda: st.apply_all(p, g, 5e-4), W, K)
    line("multi-tensor adalomo, llama-7b (1 call)", n, ms, 24)


if __name__ == "__main__":
    main()
