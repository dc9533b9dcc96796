"""ORACLE -- TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's
cpu_baseline / reference arm).  Never imported by the product package.

Two checkers:
  Restatement  oracle/_build/liborc.so  (mco_oracle.c: f64 / f32 / bf16 restatement
               of optim.cpp + the synthetic generator + ZeroPlan)
  Reference    oracle/_ref/libmco_ref.so (the unmodified reference minicollie::optim
               compiled from /root/reference by oracle/Makefile, behind ref_wrap.cpp)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "_build", "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libmco_ref.so")
REF_SRC = "/root/reference/proj"

_p, _i, _u64, _i64, _d = C.c_void_p, C.c_int, C.c_uint64, C.c_int64, C.c_double


class Config(C.Structure):
    """Same layout as mco_config / orc_config / ref_config (optim.hpp:20-35)."""

    _fields_ = [("kind", C.c_int), ("lr", C.c_double), ("weight_decay", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("beta3", C.c_double),
                ("eps", C.c_double), ("has_clip_threshold", C.c_int),
                ("clip_threshold", C.c_double), ("adalomo_clip", C.c_double),
                ("sophia_rho", C.c_double), ("update_interval", C.c_int)]

    @staticmethod
    def of(cfg) -> "Config":
        """From a paper_2312_00407_b200.optim.OptimizerConfig (or anything with its fields)."""
        if isinstance(cfg, Config):
            return cfg
        return Config(int(cfg.kind), cfg.lr, cfg.weight_decay, cfg.beta1, cfg.beta2, cfg.beta3,
                      cfg.eps, 1 if cfg.clip_threshold is not None else 0,
                      float(cfg.clip_threshold or 0.0), cfg.adalomo_clip, cfg.sophia_rho,
                      int(cfg.update_interval))


def build(ref: bool = True) -> None:
    """Build the checkers (make -C oracle).  The reference part needs /root/reference
    (present in the build container; the GPU box only uses the prebuilt .so)."""
    targets = ["oracle"] + (["ref"] if ref and os.path.isdir(REF_SRC) else [])
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_CP = C.POINTER(Config)


def _load_orc():
    lib = C.CDLL(ORC_PATH)
    sigs = {
        "orc_fmix64": (_u64, [_u64]),
        "orc_synth_key": (_u64, [_u64, C.c_uint32, C.c_uint32, C.c_uint32]),
        "orc_synth_f32": (None, [_p, _u64, _u64, _i64, _i, _i, _i]),
        "orc_synth_f64": (None, [_p, _u64, _u64, _i64, _i, _i, _i]),
        "orc_synth_bf16": (None, [_p, _u64, _u64, _i64, _i, _i, _i]),
        "orc_adamw_f64": (None, [_p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_lion_f64": (None, [_p, _p, _p, _u64, _CP, _d]),
        "orc_adan_f64": (None, [_p, _p, _p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_sophia_f64": (None, [_p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_lomo_f64": (None, [_p, _p, _u64, _d, _d]),
        "orc_sumsq_f64": (_d, [_p, _u64]),
        "orc_clip_scale": (_d, [_d, _d]),
        "orc_adalomo_f64": (None, [_p, _p, _i64, _i64, _i, _p, _p, _p, C.POINTER(_i64), _CP, _d,
                                   _d, _p]),
        "orc_adamw_f32": (None, [_p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_lion_f32": (None, [_p, _p, _p, _u64, _CP, _d]),
        "orc_adan_f32": (None, [_p, _p, _p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_sophia_f32": (None, [_p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_sophia_m64": (None, [_p, _p, _p, _p, _u64, _CP, _i64, _d]),
        "orc_lomo_f32": (None, [_p, _p, _u64, _d, _d]),
        "orc_lomo_bf16": (None, [_p, _p, _u64, _d, _d]),
        "orc_sumsq_f32": (_d, [_p, _u64]),
        "orc_sumsq_bf16": (_d, [_p, _u64]),
        "orc_f32_to_bf16": (C.c_uint16, [C.c_float]),
        "orc_bf16_to_f32": (C.c_float, [C.c_uint16]),
        "orc_zero_plan": (_i, [_u64, _i, C.POINTER(_u64), C.POINTER(_u64)]),
    }
    for n, (r, a) in sigs.items():
        f = getattr(lib, n)
        f.restype, f.argtypes = r, a
    return lib


def _load_ref():
    if not os.path.exists(REF_PATH):
        return None
    lib = C.CDLL(REF_PATH)
    sigs = {
        "ref_last_error": (C.c_char_p, []),
        "ref_parse_kind": (_i, [C.c_char_p, C.POINTER(_i)]),
        "ref_kind_name": (C.c_char_p, [_i]),
        "ref_is_fused": (_i, [_i]),
        "ref_defaults_for": (_i, [_i, _CP]),
        "ref_validate": (_i, [_CP]),
        "ref_flat_create": (_i, [_CP, C.c_size_t, C.POINTER(_p)]),
        "ref_flat_destroy": (None, [_p]),
        "ref_flat_step": (_i, [_p, _p, _p, C.c_size_t, C.c_size_t, _d]),
        "ref_flat_steps": (_i64, [_p]),
        "ref_flat_set_steps": (None, [_p, _i64]),
        "ref_flat_state_bytes": (_u64, [_p]),
        "ref_flat_num_buffers": (_i, [_p]),
        "ref_flat_buffer": (C.c_char_p, [_p, _i, C.POINTER(_p), C.POINTER(C.c_size_t)]),
        "ref_lomo_apply": (_i, [_p, _p, C.c_size_t, _d, _d]),
        "ref_lomo_fused_step": (_i, [_i, C.POINTER(_i64), C.POINTER(_p), C.POINTER(_p), _d, _d]),
        "ref_adalomo_create": (_i, [_CP, _i, C.POINTER(_i), C.POINTER(_i64), C.POINTER(_p)]),
        "ref_adalomo_destroy": (None, [_p]),
        "ref_adalomo_apply": (_i, [_p, _i, _p, _p, _d]),
        "ref_adalomo_state_bytes": (_u64, [_p]),
        "ref_state_bytes": (_i, [_i, _u64, _i, _i, _i, _i, C.POINTER(_i), C.POINTER(_i64),
                                 C.POINTER(_u64)]),
        "ref_zero_plan": (_i, [C.c_size_t, _i, _i, C.POINTER(C.c_size_t),
                               C.POINTER(C.c_size_t)]),
        "ref_bench": (_i, [_CP, _i, C.POINTER(_i), C.POINTER(_i64), _i, _i, _i, _u64, _d, _D]),
    }
    for n, (r, a) in sigs.items():
        f = getattr(lib, n)
        f.restype, f.argtypes = r, a
    return lib


if not os.path.exists(ORC_PATH):
    build(ref=True)
orc = _load_orc()
ref = _load_ref()


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def ref_check(status: int) -> None:
    if status != 0:
        raise RefError(status, ref.ref_last_error().decode())


# ---- synthetic generator (numpy views over the C restatement) ---------------------------

def synth(n: int, seed: int, role: int, tensor: int, step: int, cols: int = 0,
          scale_log2: int = 0, zero_log2: int = 0, rowcol: bool = False,
          dtype=np.float32) -> np.ndarray:
    key = orc.orc_synth_key(seed, role, tensor, step)
    if dtype == np.float32:
        out = np.empty(n, np.float32)
        orc.orc_synth_f32(_ptr(out), n, key, cols, scale_log2, zero_log2, int(rowcol))
    elif dtype == np.float64:
        out = np.empty(n, np.float64)
        orc.orc_synth_f64(_ptr(out), n, key, cols, scale_log2, zero_log2, int(rowcol))
    else:  # bf16 bit patterns
        out = np.empty(n, np.uint16)
        orc.orc_synth_bf16(_ptr(out), n, key, cols, scale_log2, zero_log2, int(rowcol))
    return out


def registry_params(shapes, seed: int, dtype=np.float32) -> list[np.ndarray]:
    """Registry-order synthetic parameters (same rule as paper_2312_00407_b200.registry)."""
    out = []
    for k, s in enumerate(shapes):
        n = int(np.prod(s))
        if len(s) == 2:
            out.append(synth(n, seed, 0, k, 0, s[1], -6, 0, False, dtype))
        else:
            out.append(np.ones(n, dtype))
    return out


def registry_grads(shapes, seed: int, step: int, dtype=np.float32) -> list[np.ndarray]:
    out = []
    for k, s in enumerate(shapes):
        n = int(np.prod(s))
        if len(s) == 2:
            out.append(synth(n, seed, 1, k, step, s[1], -7, 10, True, dtype))
        else:
            out.append(synth(n, seed, 1, k, step, 0, -7, 10, False, dtype))
    return out


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """RNE, NaN -> 0x7fff (same rule as orc_f32_to_bf16 / cvt.rn.bf16 in the kernels)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = 0x7FFF
    return r


# ---- restatement steppers ----------------------------------------------------------------

class OracleFlat:
    """FlatOptimizer restated (f64 or f32), same state layout / names as the reference."""

    NAMES = {0: ("m", "v"), 1: ("m",), 2: ("m", "v", "n", "g_prev"), 3: ("m", "h")}

    def __init__(self, cfg, n: int, dtype=np.float64):
        self.cfg = Config.of(cfg)
        self.dtype = dtype
        self.t = 0
        self.state = {name: np.zeros(n, dtype) for name in self.NAMES[self.cfg.kind]}

    def step(self, p: np.ndarray, g: np.ndarray, lr: float) -> None:
        assert p.dtype == self.dtype and g.dtype == self.dtype
        self.t += 1
        f = "f64" if self.dtype == np.float64 else "f32"
        s, c, n = self.state, C.byref(self.cfg), p.size
        k = self.cfg.kind
        if k == 0:
            getattr(orc, f"orc_adamw_{f}")(_ptr(p), _ptr(g), _ptr(s["m"]), _ptr(s["v"]), n, c,
                                          self.t, lr)
        elif k == 1:
            getattr(orc, f"orc_lion_{f}")(_ptr(p), _ptr(g), _ptr(s["m"]), n, c, lr)
        elif k == 2:
            getattr(orc, f"orc_adan_{f}")(_ptr(p), _ptr(g), _ptr(s["m"]), _ptr(s["v"]),
                                         _ptr(s["n"]), _ptr(s["g_prev"]), n, c, self.t, lr)
        elif k == 3:
            getattr(orc, f"orc_sophia_{f}")(_ptr(p), _ptr(g), _ptr(s["m"]), _ptr(s["h"]), n, c,
                                           self.t, lr)
        else:
            raise ValueError("fused kind")


class OracleSophiaM64:
    """Sophia precise-m restated (fp32 p / g / h, fp64 m and arithmetic; mco_oracle.c)."""

    def __init__(self, cfg, n: int):
        self.cfg = Config.of(cfg)
        self.t = 0
        self.state = {"m": np.zeros(n, np.float64), "h": np.zeros(n, np.float32)}

    def step(self, p: np.ndarray, g: np.ndarray, lr: float) -> None:
        assert p.dtype == np.float32 and g.dtype == np.float32
        self.t += 1
        orc.orc_sophia_m64(_ptr(p), _ptr(g), _ptr(self.state["m"]), _ptr(self.state["h"]),
                           p.size, C.byref(self.cfg), self.t, lr)


class OracleAdaLomo:
    """AdaLomoState restated in f64 (per-tensor entries, own step counters)."""

    def __init__(self, cfg, shapes):
        self.cfg = Config.of(cfg)
        self.shapes = [tuple(s) for s in shapes]
        self.entries = []
        for s in self.shapes:
            if len(s) == 2:
                self.entries.append(dict(v_row=np.zeros(s[0]), v_col=np.zeros(s[1]),
                                         v_full=np.zeros(1), t=C.c_int64(0)))
            else:
                self.entries.append(dict(v_row=np.zeros(1), v_col=np.zeros(1),
                                         v_full=np.zeros(int(np.prod(s))), t=C.c_int64(0)))

    def apply(self, k: int, p: np.ndarray, g: np.ndarray, lr: float, scale: float = 1.0):
        s, e = self.shapes[k], self.entries[k]
        fact = len(s) == 2
        R, Cc = (s[0], s[1]) if fact else (int(np.prod(s)), 1)
        scratch = np.empty(2 * p.size)
        orc.orc_adalomo_f64(_ptr(p), _ptr(np.ascontiguousarray(g, np.float64)), R, Cc,
                            int(fact), _ptr(e["v_row"]), _ptr(e["v_col"]), _ptr(e["v_full"]),
                            C.byref(e["t"]), C.byref(self.cfg), lr, scale, _ptr(scratch))


# ---- reference wrappers ------------------------------------------------------------------

class RefFlat:
    """The reference FlatOptimizer (fp64), driven through ref_wrap.cpp."""

    def __init__(self, cfg, n: int):
        h = C.c_void_p()
        ref_check(ref.ref_flat_create(C.byref(Config.of(cfg)), n, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            ref.ref_flat_destroy(self.h)
            self.h = None

    def step(self, p: np.ndarray, g: np.ndarray, lr: float) -> None:
        ref_check(ref.ref_flat_step(self.h, _ptr(p), _ptr(g), p.size, g.size, lr))

    def buffers(self) -> dict:
        out = {}
        for i in range(ref.ref_flat_num_buffers(self.h)):
            ptr, ln = C.c_void_p(), C.c_size_t()
            name = ref.ref_flat_buffer(self.h, i, C.byref(ptr), C.byref(ln)).decode()
            out[name] = np.ctypeslib.as_array(C.cast(ptr, _D), shape=(ln.value,)).copy()
        return out

    def steps(self) -> int:
        return ref.ref_flat_steps(self.h)

    def state_bytes(self) -> int:
        return ref.ref_flat_state_bytes(self.h)


class RefAdaLomo:
    def __init__(self, cfg, shapes):
        nd = (C.c_int * len(shapes))(*[len(s) for s in shapes])
        flat = [int(d) for s in shapes for d in s]
        dims = (C.c_int64 * max(len(flat), 1))(*flat)
        h = C.c_void_p()
        ref_check(ref.ref_adalomo_create(C.byref(Config.of(cfg)), len(shapes), nd, dims,
                                         C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            ref.ref_adalomo_destroy(self.h)
            self.h = None

    def apply(self, k: int, p: np.ndarray, g: np.ndarray, lr: float) -> None:
        ref_check(ref.ref_adalomo_apply(self.h, k, _ptr(p), _ptr(g), lr))

    def state_bytes(self) -> int:
        return ref.ref_adalomo_state_bytes(self.h)


def ref_lomo_fused(params: list, grads: list, lr: float, clip: float | None) -> None:
    """The reference's lomo_fused_backward_step on given grads (ref_wrap.cpp)."""
    n = len(params)
    numels = (C.c_int64 * n)(*[p.size for p in params])
    ps = (C.c_void_p * n)(*[p.ctypes.data for p in params])
    gs = (C.c_void_p * n)(*[g.ctypes.data for g in grads])
    ref_check(ref.ref_lomo_fused_step(n, numels, ps, gs, lr, -1.0 if clip is None else clip))


def ref_bench(cfg, shapes, threads: int, warmup: int, steps: int, seed: int = 2024,
              clip=None) -> float:
    """Seconds per step of the reference CPU path on `threads` host threads; clip (LOMO /
    AdaLomo): the global grad-norm pass of optim.cpp:291-303 before the updates."""
    nd = (C.c_int * len(shapes))(*[len(s) for s in shapes])
    flat = [int(d) for s in shapes for d in s]
    dims = (C.c_int64 * max(len(flat), 1))(*flat)
    out = C.c_double()
    ref_check(ref.ref_bench(C.byref(Config.of(cfg)), len(shapes), nd, dims, threads, warmup,
                            steps, seed, -1.0 if clip is None else float(clip), C.byref(out)))
    return out.value


# ---- reference arm helpers (bench.py --impl reference / cpu_baseline): the reference's
# own kind parser and defaults, no product code ------------------------------------------


def ref_config(kind: str, **overrides) -> Config:
    """OptimizerConfig::defaults_for(parse_kind(kind)) from the compiled reference
    (optim.cpp:13-61), then the given field overrides."""
    k = C.c_int()
    ref_check(ref.ref_parse_kind(kind.encode(), C.byref(k)))
    c = Config()
    ref_check(ref.ref_defaults_for(k.value, C.byref(c)))
    for a, v in overrides.items():
        setattr(c, a, v)
    return c


def llama_shapes(hidden: int, inter: int, layers: int, vocab: int, kv=None) -> list:
    """The reference registry order (model.cpp:353-370): tok_embedding, per layer
    attn_norm, q, k, v, o, mlp_norm, gate, up, down; final_norm, lm_head."""
    H, I, V, K = hidden, inter, vocab, kv or hidden
    out = [(V, H)]
    for _ in range(layers):
        out += [(H,), (H, H), (K, H), (K, H), (H, H), (H,), (I, H), (I, H), (H, I)]
    return out + [(H,), (V, H)]
