#!/usr/bin/env python3
"""One list-form AdamW step over a 350M decoder's 241 tensors and one graph-mode (DEV)
AdamW step over a 1.75 B flat slice -- the launches `ncu --set full` captures for
profiles/ncu_list_r01.md (tools/README.md)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_00407_b200 import optim  # noqa: E402
from paper_2312_00407_b200.optim import Kind, OptimizerConfig  # noqa: E402

cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
decoder = [(50304, 1024)] + [(1024, 1024)] * 4 * 24 + [(4096, 1024), (1024, 4096)] * 24 \
    + [(1024,)] * 4 * 24
ps = [torch.randn(*s, device="cuda") for s in decoder]
gs = [torch.randn(*s, device="cuda") for s in decoder]
lo = optim.FlatOptimizer(cfg, sum(p.numel() for p in ps))
lo.step_list(ps, gs, 1e-4)
torch.cuda.synchronize()
del ps, gs, lo
n = 1_750_000_000
p = torch.randn(n, device="cuda")
g = torch.randn(n, device="cuda")
gm = optim.FlatOptimizer(cfg, n)
gm.enable_graph()
gm.step(p, g, 1e-4)
torch.cuda.synchronize()
print("ok")
