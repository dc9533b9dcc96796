#!/usr/bin/env python3
"""FlatOptimizer graph mode on one B200: eager steps vs CUDA-graph replays.

(1) one AdamW step over a large flat slice: the graph-mode kernel (step scalars read
    from the device) must run at the eager kernel's speed;
(2) per-tensor optimizers (one FlatOptimizer per parameter tensor of a small model):
    eager = one host call + launch per tensor; graph = one replay of all of them;
    list = one FlatOptimizer over all tensors (mco_flat_step_list), eager and replayed.
Prints one JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_00407_b200 import optim  # noqa: E402
from paper_2312_00407_b200.optim import Kind, OptimizerConfig  # noqa: E402


def timed(fn, warm=3, it=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def capture(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    return g


def main():
    cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
    cfg.weight_decay = 0.01
    out = {}
    lr_t = torch.full((), 1e-4, dtype=torch.float64, device="cuda")

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_750_000_000
    p = torch.randn(n, device="cuda") * 0.02
    g = torch.randn(n, device="cuda") * 1e-3
    e = optim.FlatOptimizer(cfg, n)
    ms_e = timed(lambda: e.step(p, g, 1e-4), it=10)
    del e
    gm = optim.FlatOptimizer(cfg, n)
    gm.enable_graph(lr_t)
    graph = capture(lambda: gm.step(p, g, 0.0))
    ms_g = timed(graph.replay, it=10)
    out["large"] = {"n": n, "eager_ms": round(ms_e, 3), "graph_ms": round(ms_g, 3),
                    "graph_over_eager": round(ms_g / ms_e, 4)}
    del gm, graph, p, g
    torch.cuda.empty_cache()

    # per-tensor optimizers: a 350M-parameter decoder's tensors (GPU-bound) and 4000
    # small tensors (host-bound: one ctypes call + launch per tensor)
    decoder = [(50304, 1024)] + [(1024, 1024)] * 4 * 24 + [(4096, 1024), (1024, 4096)] * 24 \
        + [(1024,)] * 4 * 24
    for name, shapes in (("per_tensor_350m", decoder), ("per_tensor_small", [(16384,)] * 4000)):
        ps = [torch.randn(*s, device="cuda") * 0.02 for s in shapes]
        gs = [torch.randn(*s, device="cuda") * 1e-3 for s in shapes]
        opts = [optim.FlatOptimizer(cfg, x.numel()) for x in ps]

        def eager_all():
            for o, x, y in zip(opts, ps, gs):
                o.step(x, y, 1e-4)

        ms_e = timed(eager_all)
        for o in opts:
            o.enable_graph(lr_t)
        graph = capture(lambda: [o.step(x, y, 0.0) for o, x, y in zip(opts, ps, gs)])
        ms_g = timed(graph.replay)
        del opts, graph
        # list form: one optimizer over the flat state, the tensors stepped in place
        lo = optim.FlatOptimizer(cfg, sum(x.numel() for x in ps))
        ms_l = timed(lambda: lo.step_list(ps, gs, 1e-4))
        lo.enable_graph(lr_t)
        graph = capture(lambda: lo.step_list(ps, gs, 0.0))
        ms_lg = timed(graph.replay)
        out[name] = {"tensors": len(shapes), "params": sum(x.numel() for x in ps),
                     "eager_ms": round(ms_e, 3), "graph_ms": round(ms_g, 3),
                     "speedup": round(ms_e / ms_g, 3), "list_ms": round(ms_l, 3),
                     "list_graph_ms": round(ms_lg, 3),
                     "list_gbps": round(28 * sum(x.numel() for x in ps) / ms_l / 1e6, 1)}
        del ps, gs, lo, graph
    print(json.dumps(out))


if __name__ == "__main__":
    main()
