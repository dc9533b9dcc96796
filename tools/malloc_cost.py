#!/usr/bin/env python3
"""Cost of cudaMalloc / cudaFree of a 7B-gradient-sized buffer (27 GB) on this GPU: the
LOMO clip host path allocates its resident gradient per call."""
import time

import torch
from cuda.bindings import runtime as rt

torch.cuda.init()
for gb in (1, 8, 27):
    n = gb << 30
    t0 = time.perf_counter()
    err, ptr = rt.cudaMalloc(n)
    t1 = time.perf_counter()
    rt.cudaMemset(ptr, 0, n)
    rt.cudaDeviceSynchronize()
    t2 = time.perf_counter()
    rt.cudaFree(ptr)
    t3 = time.perf_counter()
    print(f"{gb} GiB: malloc {1e3 * (t1 - t0):.1f} ms, first touch {1e3 * (t2 - t1):.1f} ms, "
          f"free {1e3 * (t3 - t2):.1f} ms", flush=True)
