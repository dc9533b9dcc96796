"""The fp32 parity bars, in one place (north_star: within 1e-5 per element of the fp64
reference after N steps).  Every bar is |got - want| <= 1e-5 * max(|want|,
floor) per element; the floors are the smallest magnitudes fp32 arithmetic resolves
for that quantity (measured margins in DESIGN.md section 4):

  parameters  floor_i = min(RMS(p0), max(|p0_i|, lr))  -- every step computes
              p - lr * (u + wd p) with |u| <~ 1, so an element's roundings are of size
              ulp(max(|p|, lr)); elements that start or pass near 0 are held to lr.
              (Round 1 used the looser max(|want|, RMS(p0)) for every element.)
  state       floor = RMS(want) / 4 -- EMAs of sign-changing gradients (m, v of Adan)
              cancel, so near zero crossings only an absolute bar at the buffer's scale
              is attainable in fp32.
  delta p     |Δgot - Δwant| <= 1e-5 max(|Δwant_i|, N lr, N 2^-24 |p0_i| / 1e-5),
              Δ = p_N - p_0 after N steps: N lr bounds the total update (|u| <~ 1), and
              fp32 storage rounds p by up to 2^-24 |p| per step, so an update smaller
              than N 2^-24 |p0| / 1e-5 cannot be resolved to 1e-5 (norm weights = 1.0).
"""
from __future__ import annotations

import numpy as np

TOL = 1e-5


def _f64(x):
    return np.asarray(x, dtype=np.float64)


def p_err(got, want, p0, lr) -> np.ndarray:
    got, want, p0 = _f64(got), _f64(want), _f64(p0)
    rms = float(np.sqrt(np.mean(p0 ** 2)))
    floor = np.minimum(rms, np.maximum(np.abs(p0), lr))
    return np.abs(got - want) / np.maximum(np.abs(want), floor)


def state_err(got, want) -> np.ndarray:
    got, want = _f64(got), _f64(want)
    rms = float(np.sqrt(np.mean(want ** 2)))
    floor = max(rms / 4, np.finfo(np.float64).tiny)
    return np.abs(got - want) / np.maximum(np.abs(want), floor)


def dp_err(got, want, p0, lr, steps) -> np.ndarray:
    got, want, p0 = _f64(got), _f64(want), _f64(p0)
    dw = want - p0
    floor = np.maximum(steps * lr, steps * 2.0 ** -24 * np.abs(p0) / TOL)
    return np.abs((got - p0) - dw) / np.maximum(np.abs(dw), floor)


def flat_errors(got_p, want_p, p0, lr, steps, got_state=None, want_state=None) -> dict:
    """Max error of p, Δp and every named state buffer (relative to its floor)."""
    out = {"p": float(p_err(got_p, want_p, p0, lr).max()),
           "dp": float(dp_err(got_p, want_p, p0, lr, steps).max())}
    for name, w in (want_state or {}).items():
        if got_state is not None and name in got_state:
            out[name] = float(state_err(got_state[name], w).max())
    return out


def assert_flat_within(got_p, want_p, p0, lr, steps, got_state=None, want_state=None,
                       what=""):
    e = flat_errors(got_p, want_p, p0, lr, steps, got_state, want_state)
    bad = {k: v for k, v in e.items() if not v <= TOL}
    assert not bad, f"{what}: beyond 1e-5 of the fp64 reference: {bad} (all: {e})"
    return e


def exceedance(got_p, want_p, p0, lr) -> dict:
    """Fraction of elements past the parameter bar, and the largest error (Sophia's fp32
    m path is reported with these; its precise-m mode meets the bar)."""
    e = p_err(got_p, want_p, p0, lr)
    return {"fraction": float(np.mean(e > TOL)), "max_rel": float(e.max()),
            "max_abs_over_lr": float(np.max(np.abs(_f64(got_p) - _f64(want_p))) / lr)}


def record(kind: str, data: dict) -> None:
    """Merge measured errors into gpurun_out/parity.json (copied to profiles/parity.json,
    which bench.py reports beside Sophia's legs)."""
    import json
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    path = os.path.join(out, "parity.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except Exception:
        d = {}
    d[kind] = data
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
