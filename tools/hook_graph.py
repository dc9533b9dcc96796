#!/usr/bin/env python3
"""AdaLomo hook form over the 7B set: eager (one Python call per tensor, as a backward
hook issues them) vs the same 291 calls captured once into a CUDA graph and replayed --
separates the host's per-call cost from the GPU's.  Also the host time per call."""
import json
import os
import sys
import time

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
    for s in shapes:
        offs.append(offs[-1] + int(torch.tensor(s).prod()))
    views = [(p[offs[k]:offs[k + 1]], g[offs[k]:offs[k + 1]]) for k in range(len(shapes))]
    order = list(reversed(range(len(shapes))))
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    st = optim.AdaLomoState(cfg, shapes)
    s = torch.cuda.Stream()

    def hooks():
        for k in order:
            st.apply(k, views[k][0], views[k][1], 5e-4, stream=s)

    with torch.cuda.stream(s):
        for _ in range(2):
            hooks()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    K = 5
    t0 = time.perf_counter()
    ev[0].record(s)
    with torch.cuda.stream(s):
        for _ in range(K):
            hooks()
    t1 = time.perf_counter()
    ev[1].record(s)
    torch.cuda.synchronize()
    eager = ev[0].elapsed_time(ev[1]) / K
    host_us = (t1 - t0) / K / len(order) * 1e6
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        hooks()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()  # replay() launches on the current stream
    ev[0].record(cur)
    for _ in range(K):
        gr.replay()
    ev[1].record(cur)
    torch.cuda.synchronize()
    graph = ev[0].elapsed_time(ev[1]) / K
    print(json.dumps({"eager_ms": round(eager, 3), "graph_ms": round(graph, 3),
                      "host_us_per_call": round(host_us, 1), "calls": len(order)}))


if __name__ == "__main__":
    main()
