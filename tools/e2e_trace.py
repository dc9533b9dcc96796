#!/usr/bin/env python3
"""LOMO + clip through the host-span C-ABI (mco_lomo_apply_host) on pinned 7B-sized host
buffers, wall time per call; run with MCO_HOST_TRACE=1 for the per-phase split."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2312_00407_b200 import optim, registry

    n = registry.LLAMA_7B.param_count()
    hp = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hg = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hp.fill_(0.01)
    hg.fill_(1e-4)
    a, b = hp.numpy(), hg.numpy()
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        optim.lomo_step(a, b, 1e-3, clip=1.0)
        torch.cuda.synchronize()
        print(f"lomo host call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
