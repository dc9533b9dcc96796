#!/usr/bin/env python3
"""Host-side cost per call of the C-ABI entry points (wall clock, no synchronisation
inside the loop): ctypes floor, LOMO / AdaLomo hook calls on small and 7B-sized tensors."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def per_call(fn, n=400):
    import torch
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round((t1 - t0) / n * 1e6, 2)


def main():
    import torch

    from paper_2312_00407_b200 import optim
    from paper_2312_00407_b200._lib import lib
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    out = {}
    out["ctypes_kind_name"] = per_call(lambda: lib.mco_kind_name(0))
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    for shp in [(64, 64), (4096,), (4096, 4096)]:
        n = 1
        for d in shp:
            n *= d
        p = torch.zeros(n, device="cuda")
        g = torch.zeros(n, device="cuda")
        st = optim.AdaLomoState(cfg, [shp])
        out[f"adalomo_apply_{shp}"] = per_call(lambda: st.apply(0, p, g, 1e-3), 200)
        s = torch.cuda.current_stream().cuda_stream
        h = st._h
        fn = lib.mco_adalomo_apply
        pp, gp = p.data_ptr(), g.data_ptr()
        out[f"adalomo_apply_raw_{shp}"] = per_call(
            lambda: fn(h, 0, pp, 0, gp, 0, C.c_double(1e-3), None, C.c_void_p(s)), 200)
        out[f"lomo_apply_{shp}"] = per_call(lambda: optim.lomo_apply(p, g, 1e-3, 1.0), 200)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
