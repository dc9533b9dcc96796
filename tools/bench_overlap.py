#!/usr/bin/env python3
"""f4 on one B200: a training step (forward + backward + AdamW) of a deep MLP with the
optimizer either after backward (flatten-free, one FlatOptimizer step over the flat
gradient) or overlapped with backward (overlap.OverlappedZeroOptimizer: per-bucket
updates on a high-priority side stream).  Prints ms per step for both."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_00407_b200 import optim, overlap  # noqa: E402
from paper_2312_00407_b200.optim import Kind, OptimizerConfig  # noqa: E402


def mlp(width, depth):
    torch.manual_seed(0)
    layers = []
    for _ in range(depth):
        layers += [torch.nn.Linear(width, width, bias=False), torch.nn.GELU()]
    return torch.nn.Sequential(*layers).cuda()


def timed(fn, warm=3, it=10):
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


def main():
    width, depth = 4096, 24
    tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    cfg = OptimizerConfig.defaults_for(Kind.ADAMW)
    x = torch.randn(tokens, width, device="cuda")
    y = torch.randn(tokens, width, device="cuda")

    def loss_of(m):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            return ((m(x).float() - y) ** 2).mean()

    m1 = mlp(width, depth)
    params = list(m1.parameters())
    n = sum(p.numel() for p in params)
    flat_p = torch.cat([p.detach().reshape(-1) for p in params])
    flat_g = torch.zeros(n, device="cuda")
    off = 0
    for p in params:  # zero-copy flat views, as overlap.py does, so both arms match
        p.data = flat_p[off:off + p.numel()].view_as(p)
        p.grad = flat_g[off:off + p.numel()].view_as(p)
        off += p.numel()
    opt = optim.FlatOptimizer(cfg, n)

    def serial():
        flat_g.zero_()
        loss_of(m1).backward()
        opt.step(flat_p, flat_g, 1e-4)

    fwd_bwd = timed(lambda: loss_of(m1).backward())
    step_only = timed(lambda: opt.step(flat_p, flat_g, 1e-4))
    t_serial = timed(serial)
    print(f"tokens {tokens}, params {n / 1e6:.0f}M: forward+backward {fwd_bwd:.2f} ms, "
          f"AdamW step {step_only:.2f} ms, serial step {t_serial:.2f} ms")
    m2 = mlp(width, depth)
    ov = overlap.OverlappedZeroOptimizer(cfg, list(m2.parameters()), bucket_elems=1 << 24)

    def overlapped():
        ov.backward_step(lambda: loss_of(m2), 1e-4)

    t = timed(overlapped)
    print(f"  overlapped ({len(ov.buckets)} buckets): {t:.2f} ms ({t_serial - t:+.2f} ms vs serial)")


if __name__ == "__main__":
    main()
