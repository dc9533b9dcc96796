#!/usr/bin/env python3
"""Launch every hot kernel family once or twice at a bandwidth-saturating size, for
`ncu --set full` (profiles/run_ncu_r02.sh): the fp32 stored-state kinds on the TMA
pipeline (2 steps each: Adan's g_prev read starts at t = 2), Sophia precise-m, LOMO +
clip (sum of squares + update) in fp32 and bf16, AdaLomo + clip over a 2-layer 7B
subset in fp32 and bf16 (K1 .. K6), the AdaLomo hook form on one 11008 x 4096 matrix,
and the peer-memory ZeRO kernel with two virtual ranks on one device.

usage: python tools/profile_kernels.py [--elems N]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2312_00407_b200 import optim, registry
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=1 << 28)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    n = a.elems
    want = set(a.only.split(",")) if a.only else None
    torch.cuda.set_device(0)

    def on(name):
        return want is None or name in want

    def cfg(kind, **kw):
        c = OptimizerConfig.defaults_for(kind)
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    p = torch.empty(n, device="cuda")
    g = torch.empty(n, device="cuda")
    optim.synth_fill(p, 1, 0, 0, 0, 0, -6)
    optim.synth_fill(g, 1, 1, 0, 1, 0, -7, 10)
    for kind in (Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA):
        if on(kind.name.lower()):
            o = optim.FlatOptimizer(cfg(kind, weight_decay=0.01), n)
            o.step(p, g, 1e-4)
            o.step(p, g, 1e-4)
            torch.cuda.synchronize()
            del o
    if on("sophia_m64"):
        o = optim.FlatOptimizer(cfg(Kind.SOPHIA, weight_decay=0.01), n, state_dtype="f32m64")
        o.step(p, g, 1e-4)
        o.step(p, g, 1e-4)
        torch.cuda.synchronize()
        del o
    if on("lomo"):
        optim.lomo_step(p, g, 1e-3, clip=1.0)
        pb, gb = p.to(torch.bfloat16), g.to(torch.bfloat16)
        optim.lomo_step(pb, gb, 1e-3, clip=1.0)
        torch.cuda.synchronize()
        del pb, gb
    del p, g
    torch.cuda.empty_cache()
    m = registry.layer_subset(registry.LLAMA_7B, 2)
    shapes, P = m.shapes(), m.param_count()
    if on("adalomo"):
        fp = torch.empty(P, device="cuda")
        fg = torch.empty(P, device="cuda")
        registry.fill_params(fp, shapes)
        registry.fill_grads(fg, shapes, 1)
        st = optim.AdaLomoState(cfg(Kind.ADALOMO), shapes, grad_clip=1.0)
        st.apply_all(fp, fg, 5e-4)
        torch.cuda.synchronize()
        bp, bg = fp.to(torch.bfloat16), fg.to(torch.bfloat16)
        st2 = optim.AdaLomoState(cfg(Kind.ADALOMO), shapes, grad_clip=1.0)
        st2.apply_all(bp, bg, 5e-4)
        torch.cuda.synchronize()
        h = optim.AdaLomoState(cfg(Kind.ADALOMO), [(11008, 4096)])
        h.apply(0, fp[:11008 * 4096], fg[:11008 * 4096], 5e-4)
        torch.cuda.synchronize()
        del fp, fg, bp, bg, st, st2, h
    if on("peer"):
        half = 1 << 27
        world = 2
        c = cfg(Kind.ADAMW, weight_decay=0.01)
        grads = [torch.empty(half, device="cuda") for _ in range(world)]
        reps = [torch.empty(half, device="cuda") for _ in range(world)]
        for r in range(world):
            optim.synth_fill(grads[r], 1, 1, r, 1, 0, -7, 10)
            optim.synth_fill(reps[r], 1, 0, 0, 0, 0, -6)
        lo, own = 0, half // world
        o = optim.FlatOptimizer(c, own)
        o.step_peers(grads, reps, reps[0][lo:lo + own], lo, own, 1e-4)
        torch.cuda.synchronize()
    print("profile_kernels: done")


if __name__ == "__main__":
    main()
