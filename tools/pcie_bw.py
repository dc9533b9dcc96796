#!/usr/bin/env python3
"""PCIe ceiling for the e2e path: pinned H2D, D2H, and both directions at once."""
import time

import torch


def bw(fn, nbytes, it=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return nbytes * it / (time.perf_counter() - t) / 1e9


n = 1 << 30  # 4 GiB fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("H2D GB/s", round(bw(lambda: d.copy_(h, non_blocking=True), 4 * n), 1))
print("D2H GB/s", round(bw(lambda: h.copy_(d, non_blocking=True), 4 * n), 1))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print("H2D+D2H concurrent GB/s (sum)", round(bw(both, 8 * n), 1))
