#!/usr/bin/env python3
"""LOMO list form (mco_lomo_apply_list: one launch per 40 tensors) over the 7B set's 291
tensors (separate allocations), fp32 and bf16, against the flat call over one buffer."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2312_00407_b200 import optim, registry

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    shapes = registry.LLAMA_7B.shapes()
    for dt, es in ((torch.float32, 4), (torch.bfloat16, 2)):
        ps = [torch.empty(s, device="cuda", dtype=dt).normal_(0, 0.02) for s in shapes]
        gs = [torch.empty(s, device="cuda", dtype=dt).normal_(0, 1e-3) for s in shapes]
        n = sum(p.numel() for p in ps)

        def run():
            optim.lomo_apply_list(ps, gs, 1e-3, 1.0)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(json.dumps({"dtype": str(dt).split(".")[-1], "tensors": len(ps), "ms": round(ms, 3),
                          "frac": round(3 * es * n / (ms * 1e-3) / 1e9 / peak, 4)}), flush=True)
        del ps, gs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
