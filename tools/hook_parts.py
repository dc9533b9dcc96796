#!/usr/bin/env python3
"""Where the AdaLomo hook form's time goes over the 7B set: the 291 per-tensor calls in
backward order, the same calls without the 1-D tensors, the 1-D tensors alone, and the
matrices by shape -- each captured once into a CUDA graph and replayed (GPU time only).

usage: python tools/hook_parts.py   (env knobs of adalomo.cu apply, e.g. MCO_ADALOMO_SMALL)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
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
    for sh in shapes:
        offs.append(offs[-1] + int(torch.tensor(sh).prod()))
    views = [(p[offs[k]:offs[k + 1]], g[offs[k]:offs[k + 1]]) for k in range(len(shapes))]
    order = list(reversed(range(len(shapes))))
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    st = optim.AdaLomoState(cfg, shapes)
    s = torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def graph_ms(ks, K=5):
        def run():
            for k in ks:
                st.apply(k, views[k][0], views[k][1], 5e-4, stream=s)
        with torch.cuda.stream(s):
            run()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            run()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        gr.replay()
        ev[0].record(cur)
        for _ in range(K):
            gr.replay()
        ev[1].record(cur)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / K

    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("MCO_")}}
    out["all_ms"] = graph_ms(order)
    mats = [k for k in order if len(shapes[k]) == 2]
    vecs = [k for k in order if len(shapes[k]) == 1]
    out["matrices_ms"] = graph_ms(mats)
    out["vectors_ms"] = graph_ms(vecs)
    out["n_vectors"] = len(vecs)
    by = {}
    for k in mats:
        by.setdefault(tuple(shapes[k]), []).append(k)
    for sh, ks in by.items():
        ms = graph_ms(ks)
        elems = sh[0] * sh[1]
        out["x".join(map(str, sh))] = {"calls": len(ks), "us_per_call": round(ms * 1e3 / len(ks), 2),
                                       "floor_us": round(24 * elems / 6434.2e3, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
