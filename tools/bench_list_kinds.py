#!/usr/bin/env python3
"""List form over a 350M decoder's 241 tensors, every stored-state kind (one B200):
ms per step and the fraction of the measured copy bandwidth (algorithmic bytes)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_00407_b200 import optim  # noqa: E402
from paper_2312_00407_b200.optim import Kind, OptimizerConfig  # noqa: E402

BYTES = {Kind.ADAMW: 28, Kind.LION: 20, Kind.ADAN: 44, Kind.SOPHIA: 24}
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


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


decoder = [(50304, 1024)] + [(1024, 1024)] * 4 * 24 + [(4096, 1024), (1024, 4096)] * 24 \
    + [(1024,)] * 4 * 24
ps = [torch.randn(*s, device="cuda") * 0.02 for s in decoder]
gs = [torch.randn(*s, device="cuda") * 1e-3 for s in decoder]
n = sum(p.numel() for p in ps)
out = {}
for kind, nb in BYTES.items():
    cfg = OptimizerConfig.defaults_for(kind)
    cfg.update_interval = 1 << 30  # Sophia: non-refresh steps (24 B/param)
    opt = optim.FlatOptimizer(cfg, n)
    opt.step_list(ps, gs, 1e-4)  # t = 1 (Adan's first step reads no g_prev)
    ms = timed(lambda: opt.step_list(ps, gs, 1e-4))
    out[kind.name.lower()] = {"ms": round(ms, 4), "frac": round(nb * n / ms / 1e6 / PEAK, 4)}
    del opt
print(json.dumps({"tensors": len(decoder), "params": n, "list": out}))
