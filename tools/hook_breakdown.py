#!/usr/bin/env python3
"""Where the AdaLomo hook form's time goes, per tensor shape of the 7B set: one
AdaLomoState per shape, the hook call (apply, fused: 5 launches) repeated, and the three
phases (mco_adalomo_phase, unfused: 7 launches) repeated one at a time, each against its
traffic floor at the measured copy bandwidth.  CUDA events, after warm-up."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2312_00407_b200 import optim
    from paper_2312_00407_b200.optim import Kind, OptimizerConfig

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    R = int(os.environ.get("HB_R", "20"))

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(R):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / R * 1e3  # us

    shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (32000, 4096), (4096,)]
    for dt in (torch.float32, torch.bfloat16):
        es = 4 if dt == torch.float32 else 2
        for s in shapes:
            n = 1
            for d in s:
                n *= d
            p = (torch.randn(n, device="cuda") * 0.02).to(dt)
            g = (torch.randn(n, device="cuda") * 1e-3).to(dt)
            st = optim.AdaLomoState(cfg, [s])
            hook = timed(lambda: st.apply(0, p, g, 1e-3))
            ph = [timed(lambda i=i: st.phase(i, p, g, 1e-3)) for i in (1, 2, 3)]
            fl = [n * es * 2 / peak / 1e3, n * es / peak / 1e3, n * es * 3 / peak / 1e3]
            print(json.dumps({"dtype": str(dt).split(".")[-1], "shape": list(s),
                              "hook_us": round(hook, 1), "floor_us": round(sum(fl), 1),
                              "frac": round(sum(fl) / hook, 3),
                              "phase_us": [round(x, 1) for x in ph],
                              "phase_floor_us": [round(x, 1) for x in fl]}), flush=True)
            del st, p, g


if __name__ == "__main__":
    main()
