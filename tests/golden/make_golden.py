#!/usr/bin/env python3
"""Generate tests/golden/reference_vectors.npz from the REFERENCE ITSELF
(oracle/_ref/libmco_ref.so = minicollie::optim compiled from /root/reference).

Inputs are the counter-based synthetic generator (exact fp64 values); outputs are
what the reference's FlatOptimizer / lomo_apply / lomo_fused_backward_step /
AdaLomoState::apply / ZeroPlan produce.  The fixtures let the parity tests run
where /root/reference is absent, and pin the oracle restatement independently.

usage: python tests/golden/make_golden.py     (needs oracle/_ref built)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import oracle as O  # noqa: E402
from paper_2312_00407_b200.optim import Kind, OptimizerConfig  # noqa: E402

N, STEPS, LR = 1031, 5, 1e-3
ADA_SHAPES = [(6, 9), (7,), (33, 17)]


def main():
    assert O.ref is not None, "build oracle/_ref first (make -C oracle ref)"
    out = {}
    p0 = O.synth(N, 77, 0, 0, 0, 0, -6, 0, False, np.float64)
    out["flat_p0"] = p0
    for t in range(1, STEPS + 1):
        out[f"flat_g{t}"] = O.synth(N, 77, 1, 0, t, 0, -7, 10, False, np.float64)
    for kind in (Kind.ADAMW, Kind.LION, Kind.ADAN, Kind.SOPHIA):
        cfg = OptimizerConfig.defaults_for(kind)
        cfg.weight_decay = 0.01
        cfg.update_interval = 2
        r, p = O.RefFlat(cfg, N), p0.copy()
        for t in range(1, STEPS + 1):
            r.step(p, out[f"flat_g{t}"], LR)
        out[f"{kind.name.lower()}_p"] = p
        for name, buf in r.buffers().items():
            out[f"{kind.name.lower()}_{name}"] = buf
    # LOMO two-pass clip (lomo_fused_backward_step) over three tensors
    sizes = [100, 7, 300]
    ps = [O.synth(n, 78, 0, k, 0, 0, -6, 0, False, np.float64) for k, n in enumerate(sizes)]
    gs = [O.synth(n, 78, 1, k, 1, 0, -2, 0, False, np.float64) for k, n in enumerate(sizes)]
    out["lomo_p0"], out["lomo_g"] = np.concatenate(ps), np.concatenate(gs)
    O.ref_lomo_fused(ps, gs, 0.1, 0.5)
    out["lomo_clip_p"] = np.concatenate(ps)
    # AdaLomo, 3 steps
    cfg = OptimizerConfig.defaults_for(Kind.ADALOMO)
    r = O.RefAdaLomo(cfg, ADA_SHAPES)
    aps = [O.synth(int(np.prod(s)), 79, 0, k, 0, 0, -3, 0, False, np.float64)
           for k, s in enumerate(ADA_SHAPES)]
    out["adalomo_p0"] = np.concatenate(aps)
    for t in range(1, 4):
        ags = [O.synth(int(np.prod(s)), 79, 1, k, t, 0, -5, 4, False, np.float64)
               for k, s in enumerate(ADA_SHAPES)]
        out[f"adalomo_g{t}"] = np.concatenate(ags)
        for k in range(len(ADA_SHAPES)):
            r.apply(k, aps[k], ags[k], 5e-3)
    out["adalomo_p"] = np.concatenate(aps)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                     "reference_vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
