"""Host-side mirror of the reference optimizer API, ``minicollie::optim``
(/root/reference/proj/core/include/minicollie/optim.hpp), over the C-ABI.

Same names, argument meaning and error behaviour as the reference:

    Kind, parse_kind, kind_name, is_fused          optim.hpp:14-18
    OptimizerConfig.defaults_for / validate         optim.hpp:20-35
    FlatOptimizer(cfg, owned_len).step(p, g, lr)    optim.hpp:40-64
    lomo_apply(param, grad, lr, scale)              optim.hpp:71
    AdaLomoState(cfg, shapes).apply(i, p, g, lr)    optim.hpp:76-96
    PrecisionPolicy, state_bytes                    optim.hpp:113-127

Device path: torch CUDA tensors (stream-ordered on torch's current stream).
Host path (the reference's ``std::span<double>`` overload): numpy arrays, staged
through the device by ``mco_flat_step_host``.  Every update runs in the sm_100a
kernels of ``csrc/``; there is no CPU implementation here.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import MCO_BF16, MCO_F32, MCO_F32M64, MCO_F64, lib

# ---- errors (errors.hpp:11-32) ------------------------------------------------------


class MinicollieError(RuntimeError):
    status = -1


class ConfigError(MinicollieError):
    status = _lib.MCO_CONFIG


class DataError(MinicollieError):
    status = _lib.MCO_DATA


class ContractError(MinicollieError):
    status = _lib.MCO_CONTRACT


class ProtocolError(MinicollieError):
    status = _lib.MCO_PROTOCOL


class IoError(MinicollieError):
    status = _lib.MCO_IO


class CudaError(MinicollieError):
    status = _lib.MCO_CUDA


_ERRORS = {c.status: c for c in (ConfigError, DataError, ContractError, ProtocolError, IoError,
                                 CudaError)}


def _check(status: int) -> None:
    if status != _lib.MCO_OK:
        msg = lib.mco_last_error().decode()
        raise _ERRORS.get(status, MinicollieError)(msg)


# ---- kinds / config -------------------------------------------------------------------


class Kind(enum.IntEnum):
    """optim.hpp:14"""

    ADAMW = 0
    LION = 1
    ADAN = 2
    SOPHIA = 3
    LOMO = 4
    ADALOMO = 5


def parse_kind(name: str) -> Kind:
    out = C.c_int()
    _check(lib.mco_parse_kind(name.encode(), C.byref(out)))
    return Kind(out.value)


def kind_name(kind: int) -> str:
    s = lib.mco_kind_name(int(kind))
    if s is None:
        raise ConfigError("unknown optimizer kind")
    return s.decode()


def is_fused(kind: int) -> bool:
    return bool(lib.mco_is_fused(int(kind)))


@dataclass
class OptimizerConfig:
    """optim.hpp:20-35; defaults as the reference's struct initialisers."""

    kind: Kind = Kind.ADAMW
    lr: float = 1e-3
    weight_decay: float = 0.0
    beta1: float = 0.9
    beta2: float = 0.999
    beta3: float = 0.99
    eps: float = 1e-8
    clip_threshold: Optional[float] = None
    adalomo_clip: float = 1.0
    sophia_rho: float = 0.04
    update_interval: int = 10

    @staticmethod
    def defaults_for(kind: int) -> "OptimizerConfig":
        c = _lib.mco_config()
        _check(lib.mco_defaults_for(int(kind), C.byref(c)))
        return OptimizerConfig._from_c(c)

    def validate(self) -> None:
        _check(lib.mco_validate(C.byref(self._to_c())))

    def _to_c(self) -> _lib.mco_config:
        return _lib.mco_config(
            int(self.kind), self.lr, self.weight_decay, self.beta1, self.beta2, self.beta3,
            self.eps, 1 if self.clip_threshold is not None else 0,
            float(self.clip_threshold or 0.0), self.adalomo_clip, self.sophia_rho,
            int(self.update_interval))

    @staticmethod
    def _from_c(c: _lib.mco_config) -> "OptimizerConfig":
        return OptimizerConfig(
            Kind(c.kind), c.lr, c.weight_decay, c.beta1, c.beta2, c.beta3, c.eps,
            c.clip_threshold if c.has_clip_threshold else None, c.adalomo_clip, c.sophia_rho,
            c.update_interval)


@dataclass
class PrecisionPolicy:
    """optim.hpp:113-119"""

    param_dtype_bytes: int = 2
    grad_dtype_bytes: int = 4
    master_copy: bool = True

    def needs_master(self) -> bool:
        return self.master_copy and self.param_dtype_bytes < 4


def _shape_arrays(shapes: Sequence[Sequence[int]]):
    nd = (C.c_int * max(len(shapes), 1))(*[len(s) for s in shapes])
    flat = [int(d) for s in shapes for d in s]
    dims = (C.c_int64 * max(len(flat), 1))(*flat)
    return nd, dims


def state_bytes(kind: int, param_count: int, policy: PrecisionPolicy,
                shapes: Sequence[Sequence[int]] = ()) -> int:
    """optim.hpp:124-127 / optim.cpp:339-362"""
    nd, dims = _shape_arrays(shapes)
    out = C.c_uint64()
    _check(lib.mco_state_bytes(int(kind), int(param_count), policy.param_dtype_bytes,
                               policy.grad_dtype_bytes, int(policy.master_copy), len(shapes),
                               nd, dims, C.byref(out)))
    return out.value


# ---- tensor plumbing (torch for device memory / streams only) ---------------------------


def _torch():
    import torch

    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return MCO_F32
    if t.dtype == torch.bfloat16:
        return MCO_BF16
    if t.dtype == torch.float64:
        return MCO_F64
    raise ContractError(f"unsupported dtype {t.dtype}")


def _np_dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return MCO_F32
    if a.dtype == np.float64:
        return MCO_F64
    raise ContractError(f"unsupported host dtype {a.dtype}")


def _dev(t, what: str):
    if not t.is_cuda:
        raise ContractError(f"{what}: expected a CUDA tensor")
    if not t.is_contiguous():
        raise ContractError(f"{what}: expected a contiguous tensor")
    return t


def _device(device: Optional[int]) -> int:
    """Explicit device index, or the calling thread's current CUDA device (one process
    per GPU: rank r works on cuda:r after torch.cuda.set_device)."""
    if device is not None:
        return int(device)
    torch = _torch()
    # no CUDA device: 0 (host-side argument checks still run; device work fails loudly)
    return int(torch.cuda.current_device()) if torch.cuda.is_available() else 0


def _stream(stream) -> int:
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    _TYPESTR = {MCO_F32: "<f4", MCO_F64: "<f8"}

    def __init__(self, ptr: int, n: int, dtype: int, owner):
        self._owner = owner  # keeps the handle (and its allocation) alive
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": self._TYPESTR[dtype], "data": (int(ptr), False),
            "version": 3, "strides": None, "stream": None}


def _as_tensor(ptr: int, n: int, dtype: int, owner, device: int):
    torch = _torch()
    return torch.as_tensor(_CudaArray(ptr, n, dtype, owner), device=f"cuda:{device}")


# ---- FlatOptimizer ----------------------------------------------------------------------


class FlatOptimizer:
    """optim.hpp:40-64: element-wise optimizer over a flat owned slice.

    state_dtype: "f32" (product path), "f64" (bit-exact parity mode) or, Sophia only,
    "f32m64" (precise-m: fp64 first moment and fp64 per-element arithmetic on fp32
    params / h, within 1e-5 per element of the fp64 reference where fp32 m is not).
    """

    def __init__(self, cfg: OptimizerConfig, owned_len: int, device: Optional[int] = None,
                 state_dtype: str = "f32"):
        self._cfg = cfg
        self._n = int(owned_len)
        self._sd = {"f32": MCO_F32, "f64": MCO_F64, "f32m64": MCO_F32M64}[state_dtype]
        h = C.c_void_p()
        self.device = _device(device)
        self._destroy = lib.mco_flat_destroy  # kept: module globals vanish at shutdown
        _check(lib.mco_flat_create(C.byref(cfg._to_c()), self._n, self.device, self._sd,
                                   C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._destroy(h)
            self._h = None

    def step(self, params, grads, lr: float, stream=None) -> None:
        """FlatOptimizer::step (optim.cpp:100-112).  torch CUDA tensors -> device
        path; numpy arrays -> the host-span overload (synchronous)."""
        if isinstance(params, np.ndarray):
            if not (params.flags.c_contiguous and grads.flags.c_contiguous):
                raise ContractError("step: host arrays must be contiguous")
            _check(lib.mco_flat_step_host(
                self._h, params.ctypes.data, _np_dtype_code(params), params.size,
                grads.ctypes.data, _np_dtype_code(grads), grads.size, float(lr)))
            return
        _dev(params, "step params")
        _dev(grads, "step grads")
        _check(lib.mco_flat_step(self._h, params.data_ptr(), _dtype_code(params),
                                 params.numel(), grads.data_ptr(), _dtype_code(grads),
                                 grads.numel(), float(lr), _stream(stream)))

    def step_list(self, params, grads, lr: float, stream=None) -> None:
        """List form (mco_flat_step_list): params[i] / grads[i] are separate contiguous
        CUDA tensors (e.g. a model's parameters and their .grad) in registry order; the
        state is the flat slice the flattened vector would give each tensor, so this
        equals step() over the concatenation bit for bit, without flattening."""
        params, grads = list(params), list(grads)
        n = len(params)
        if n != len(grads):
            raise ContractError("step_list: params / grads length mismatch")
        for i, (p, g) in enumerate(zip(params, grads)):
            _dev(p, "step_list param")
            _dev(g, "step_list grad")
            if p.numel() != g.numel():
                raise ContractError(f"step_list: tensor {i}: {p.numel()} params vs "
                                    f"{g.numel()} grads")
            if not (p.is_contiguous() and g.is_contiguous()):
                raise ContractError(f"step_list: tensor {i} is not contiguous")
        if n == 0:
            pd = gd = MCO_F32 if self._sd == MCO_F32 else MCO_F64
        else:
            pd, gd = _dtype_code(params[0]), _dtype_code(grads[0])
            if any(_dtype_code(p) != pd for p in params) or any(
                    _dtype_code(g) != gd for g in grads):
                raise ContractError("step_list: mixed dtypes in one list")
        pt = (C.c_void_p * max(n, 1))(*[p.data_ptr() for p in params])
        gt = (C.c_void_p * max(n, 1))(*[g.data_ptr() for g in grads])
        lt = (C.c_uint64 * max(n, 1))(*[p.numel() for p in params])
        _check(lib.mco_flat_step_list(self._h, n, pt, pd, gt, gd, lt, float(lr),
                                      _stream(stream)))

    def step_mixed(self, master, grads, param_out, lr: float, stream=None) -> None:
        """fp32 master step that also writes the bf16 parameter copy."""
        _dev(master, "master")
        _dev(grads, "grads")
        _dev(param_out, "param_out")
        if master.numel() != grads.numel() or param_out.numel() != master.numel():
            raise ContractError(
                f"optimizer step: params/grads length mismatch: {master.numel()} vs "
                f"{grads.numel()}")
        _check(lib.mco_flat_step_mixed(self._h, master.data_ptr(), grads.data_ptr(),
                                       _dtype_code(grads), param_out.data_ptr(),
                                       master.numel(), float(lr), _stream(stream)))

    def steps_taken(self) -> int:
        t = C.c_int64()
        _check(lib.mco_flat_get_steps(self._h, C.byref(t)))
        return t.value

    def set_steps_taken(self, t: int) -> None:
        _check(lib.mco_flat_set_steps(self._h, int(t)))

    def enable_graph(self, lr=None) -> None:
        """CUDA-graph mode (mco_flat_graph_enable): the step counter and the step
        scalars move to the device, so ``step`` can be captured into a
        torch.cuda.CUDAGraph and each replay is the next step (bit-identical to eager).
        ``lr``: optional 0-dim float64 CUDA tensor read at every step (update it between
        replays for a schedule); None = the lr passed to each captured call."""
        ptr = None
        if lr is not None:
            if lr.dtype != _torch().float64 or lr.numel() != 1 or not lr.is_cuda:
                raise ContractError("enable_graph: lr must be a 1-element float64 CUDA tensor")
            self._graph_lr = lr  # keep it alive while the library reads it
            ptr = lr.data_ptr()
        _check(lib.mco_flat_graph_enable(self._h, ptr))

    def disable_graph(self) -> None:
        _check(lib.mco_flat_graph_disable(self._h))
        self._graph_lr = None

    def state_bytes_runtime(self) -> int:
        out = C.c_uint64()
        _check(lib.mco_flat_state_bytes(self._h, C.byref(out)))
        return out.value

    def buffers(self):
        """[(name, device tensor view)] in the reference order m, v, n, h, g_prev."""
        nb = C.c_int()
        _check(lib.mco_flat_num_buffers(self._h, C.byref(nb)))
        out = []
        for i in range(nb.value):
            name, ptr, ln, dt = C.c_char_p(), C.c_void_p(), C.c_uint64(), C.c_int()
            _check(lib.mco_flat_buffer(self._h, i, C.byref(name), C.byref(ptr), C.byref(ln),
                                       C.byref(dt)))
            out.append((name.value.decode(),
                        _as_tensor(ptr.value, ln.value, dt.value, self, self.device)))
        return out

    def config(self) -> OptimizerConfig:
        return self._cfg

    def step_peers(self, grad_bufs, param_bufs, master, offset: int, n: int, lr: float,
                   grad_dtype=None, param_dtype=None, stream=None) -> None:
        """ZeRO step fused with reduce-scatter / all-gather over peer memory
        (mco_flat_step_peers).  grad_bufs / param_bufs: device pointers (ints) or
        CUDA tensors of every rank's flat buffers, this device's view of them."""
        def ptr(x):
            return x.data_ptr() if hasattr(x, "data_ptr") else int(x)

        npeers = len(grad_bufs)
        gd = grad_dtype if grad_dtype is not None else _dtype_code(grad_bufs[0])
        pd = param_dtype if param_dtype is not None else _dtype_code(param_bufs[0])
        ga = (C.c_void_p * npeers)(*[ptr(x) for x in grad_bufs])
        pa = (C.c_void_p * npeers)(*[ptr(x) for x in param_bufs])
        _check(lib.mco_flat_step_peers(self._h, ga, gd, pa, pd, npeers, ptr(master), int(offset),
                                       int(n), float(lr), _stream(stream)))


# ---- LOMO -------------------------------------------------------------------------------


def lomo_apply(param, grad, lr: float, scale: float = 1.0, stream=None) -> None:
    """optim.cpp:185-190: param -= (lr*scale) * grad (in place).  numpy (host)
    arrays go through the pipelined host path (mco_lomo_apply_host)."""
    if isinstance(param, np.ndarray):
        _check(lib.mco_lomo_apply_host(param.ctypes.data, _np_dtype_code(param),
                                       grad.ctypes.data, _np_dtype_code(grad), param.size,
                                       float(lr), float(scale), -1.0))
        return
    _dev(param, "lomo param")
    _dev(grad, "lomo grad")
    if param.numel() != grad.numel():
        raise ContractError("lomo_apply: param/grad length mismatch")
    _check(lib.mco_lomo_apply(param.data_ptr(), _dtype_code(param), grad.data_ptr(),
                              _dtype_code(grad), param.numel(), float(lr), float(scale),
                              _stream(stream)))


def lomo_apply_clipped(param, grad, lr: float, grad_sumsq, clip: float, stream=None) -> None:
    """lomo_apply with scale = clip/||g|| iff ||g|| > clip (optim.cpp:302-303),
    ||g||^2 read from the device scalar `grad_sumsq` (float64 CUDA tensor)."""
    _dev(param, "lomo param")
    _dev(grad, "lomo grad")
    _check(lib.mco_lomo_apply_clipped(param.data_ptr(), _dtype_code(param), grad.data_ptr(),
                                      _dtype_code(grad), param.numel(), float(lr),
                                      grad_sumsq.data_ptr(), float(clip), _stream(stream)))


def lomo_apply_list(params, grads, lr: float, scale: float = 1.0, grad_sumsq=None,
                    clip: Optional[float] = None, stream=None) -> None:
    """lomo_apply over separate CUDA tensors in one launch per 40 tensors
    (mco_lomo_apply_list), each tensor's update bit-identical to lomo_apply's; with
    grad_sumsq (float64 CUDA scalar) and clip: the global-norm clip rule as
    lomo_apply_clipped."""
    params, grads = list(params), list(grads)
    n = len(params)
    if n != len(grads):
        raise ContractError("lomo_apply_list: params / grads length mismatch")
    if n == 0:
        return
    for i, (p, g) in enumerate(zip(params, grads)):
        _dev(p, "lomo param")
        _dev(g, "lomo grad")
        if p.numel() != g.numel():
            raise ContractError(f"lomo_apply_list: tensor {i}: param/grad length mismatch")
        if not (p.is_contiguous() and g.is_contiguous()):
            raise ContractError(f"lomo_apply_list: tensor {i} is not contiguous")
    pd, gd = _dtype_code(params[0]), _dtype_code(grads[0])
    if any(_dtype_code(p) != pd for p in params) or any(_dtype_code(g) != gd for g in grads):
        raise ContractError("lomo_apply_list: mixed dtypes in one list")
    if (grad_sumsq is None) != (clip is None):
        raise ContractError("lomo_apply_list: grad_sumsq and clip go together")
    pt = (C.c_void_p * n)(*[p.data_ptr() for p in params])
    gt = (C.c_void_p * n)(*[g.data_ptr() for g in grads])
    lt = (C.c_uint64 * n)(*[p.numel() for p in params])
    _check(lib.mco_lomo_apply_list(n, pt, pd, gt, gd, lt, float(lr), float(scale),
                                   grad_sumsq.data_ptr() if grad_sumsq is not None else None,
                                   float(clip) if clip is not None else 0.0, _stream(stream)))


def sumsq(x, out=None, accumulate: bool = False, stream=None):
    """Deterministic sum of squares into a float64 CUDA scalar (optim.cpp:294-300)."""
    torch = _torch()
    _dev(x, "sumsq input")
    if out is None:
        out = torch.zeros((), dtype=torch.float64, device=x.device)
    _check(lib.mco_sumsq(x.data_ptr(), _dtype_code(x), x.numel(), out.data_ptr(),
                         int(accumulate), _stream(stream)))
    return out


def lomo_step(params, grads, lr: float, clip: Optional[float] = None, stream=None,
              grad_sumsq=None):
    """Flat-buffer form of lomo_fused_backward_step (optim.cpp:284-318): with a
    clip, one sum-of-squares pass then the scaled update; otherwise one pass.
    `grad_sumsq` lets a caller supply an already all-reduced device norm^2.
    numpy (host) arrays: pipelined through the device (mco_lomo_apply_host)."""
    if isinstance(params, np.ndarray):
        _check(lib.mco_lomo_apply_host(params.ctypes.data, _np_dtype_code(params),
                                       grads.ctypes.data, _np_dtype_code(grads), params.size,
                                       float(lr), 1.0, -1.0 if clip is None else float(clip)))
        return None
    if clip is None:
        lomo_apply(params, grads, lr, 1.0, stream)
        return None
    if grad_sumsq is None:
        grad_sumsq = sumsq(grads, stream=stream)
    lomo_apply_clipped(params, grads, lr, grad_sumsq, clip, stream)
    return grad_sumsq


# ---- AdaLomo -------------------------------------------------------------------------------


class AdaLomoState:
    """optim.hpp:76-96.  `shapes` in registry order; 2-D -> factored."""

    def __init__(self, cfg: OptimizerConfig, shapes: Sequence[Sequence[int]],
                 device: Optional[int] = None, grad_clip: Optional[float] = None):
        """grad_clip: opt-in global grad-norm clip of the gradients (BASELINE C3; the
        reference's AdaLomoState ignores cfg.clip_threshold, which is LOMO's field,
        optim.hpp:28) -- the LOMO rule, optim.cpp:302-303, applied to g first."""
        self._cfg = cfg
        self.grad_clip = grad_clip
        self.shapes = [tuple(int(d) for d in s) for s in shapes]
        self.numels = [int(np.prod(s)) if len(s) else 1 for s in self.shapes]
        self.offsets = np.concatenate([[0], np.cumsum(self.numels)]).astype(np.int64)
        nd, dims = _shape_arrays(self.shapes)
        h = C.c_void_p()
        self.device = _device(device)
        self._destroy = lib.mco_adalomo_destroy
        _check(lib.mco_adalomo_create(C.byref(cfg._to_c()), len(self.shapes), nd, dims,
                                      self.device, C.byref(h)))
        self._h = h
        if grad_clip is not None:
            _check(lib.mco_adalomo_set_grad_clip(h, 1, float(grad_clip)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._destroy(h)
            self._h = None

    def apply(self, index: int, param, grad, lr: float, grad_sumsq=None, stream=None) -> None:
        """AdaLomoState::apply (optim.cpp:215-275) for tensor `index` (hook form)."""
        _dev(param, "adalomo param")
        _dev(grad, "adalomo grad")
        if not (0 <= index < len(self.shapes)) or param.numel() != self.numels[index]:
            raise ContractError(f"adalomo: unknown parameter '{index}'")
        _check(lib.mco_adalomo_apply(
            self._h, int(index), param.data_ptr(), _dtype_code(param), grad.data_ptr(),
            _dtype_code(grad), float(lr),
            grad_sumsq.data_ptr() if grad_sumsq is not None else None, _stream(stream)))

    def apply_list(self, first: int, params, grads, lr: float, grad_sumsq=None,
                   stream=None) -> None:
        """Hook form for consecutive tensors first, first+1, ...: params[i] / grads[i]
        are tensor first+i (separate CUDA tensors).  == len(params) apply() calls."""
        params, grads = list(params), list(grads)
        n = len(params)
        if n != len(grads):
            raise ContractError("adalomo apply_list: params / grads length mismatch")
        if n == 0:
            return
        for i, (p, g) in enumerate(zip(params, grads)):
            _dev(p, "adalomo param")
            _dev(g, "adalomo grad")
            k = first + i
            if not (0 <= k < len(self.shapes)) or p.numel() != self.numels[k]:
                raise ContractError(f"adalomo: unknown parameter '{k}'")
        pt = (C.c_void_p * n)(*[p.data_ptr() for p in params])
        gt = (C.c_void_p * n)(*[g.data_ptr() for g in grads])
        _check(lib.mco_adalomo_apply_list(
            self._h, int(first), int(first) + n, pt, _dtype_code(params[0]), gt,
            _dtype_code(grads[0]), float(lr),
            grad_sumsq.data_ptr() if grad_sumsq is not None else None, _stream(stream)))

    def apply_all(self, flat_params, flat_grads, lr: float, stream=None) -> None:
        """Every tensor in one multi-tensor pass over registry-order flat buffers;
        global grad-norm clip when the state was built with grad_clip.  numpy (host) arrays:
        per-tensor H2D / apply / D2H pipeline (mco_adalomo_apply_all_host)."""
        if isinstance(flat_params, np.ndarray):
            if flat_params.size != int(self.offsets[-1]) or flat_grads.size != flat_params.size:
                raise ContractError("adalomo: flat buffer length does not match the registry")
            _check(lib.mco_adalomo_apply_all_host(
                self._h, flat_params.ctypes.data, _np_dtype_code(flat_params),
                flat_grads.ctypes.data, _np_dtype_code(flat_grads), float(lr)))
            return
        _dev(flat_params, "adalomo params")
        _dev(flat_grads, "adalomo grads")
        if flat_params.numel() != int(self.offsets[-1]) or flat_grads.numel() != int(
                self.offsets[-1]):
            raise ContractError("adalomo: flat buffer length does not match the registry")
        _check(lib.mco_adalomo_apply_all(self._h, flat_params.data_ptr(),
                                         _dtype_code(flat_params), flat_grads.data_ptr(),
                                         _dtype_code(flat_grads), float(lr), _stream(stream)))

    def state_bytes_runtime(self) -> int:
        out = C.c_uint64()
        _check(lib.mco_adalomo_state_bytes(self._h, C.byref(out)))
        return out.value

    # ---- row-split sharding (csrc: mco_adalomo_set_shard / _phase / _payload) ----
    def set_shard(self, index: int, global_rows: int, weight: float) -> None:
        _check(lib.mco_adalomo_set_shard(self._h, int(index), int(global_rows), float(weight)))

    def phase(self, phase: int, flat_params, flat_grads, lr: float, stream=None) -> None:
        _dev(flat_params, "adalomo params")
        _dev(flat_grads, "adalomo grads")
        _check(lib.mco_adalomo_phase(self._h, int(phase), flat_params.data_ptr(),
                                     _dtype_code(flat_params), flat_grads.data_ptr(),
                                     _dtype_code(flat_grads), float(lr), _stream(stream)))

    def payload(self, which: int):
        """fp64 device view of the statistics (0) or sum-u^2 (1) payload."""
        ptr, ln = C.c_void_p(), C.c_uint64()
        _check(lib.mco_adalomo_payload(self._h, int(which), C.byref(ptr), C.byref(ln)))
        return _as_tensor(ptr.value, ln.value, MCO_F64, self, self.device)

    def steps(self, index: int) -> int:
        t = C.c_int64()
        _check(lib.mco_adalomo_get_steps(self._h, int(index), C.byref(t)))
        return t.value

    def buffer(self, index: int, which: str):
        """fp64 device view of v_row / v_col / v_full for tensor `index` (None if absent)."""
        w = {"v_row": 0, "v_col": 1, "v_full": 2}[which]
        ptr, ln = C.c_void_p(), C.c_uint64()
        _check(lib.mco_adalomo_buffer(self._h, int(index), w, C.byref(ptr), C.byref(ln)))
        if not ptr.value:
            return None
        return _as_tensor(ptr.value, ln.value, MCO_F64, self, self.device)


# ---- misc ---------------------------------------------------------------------------------


def zero_plan(total_len: int, dp_size: int, stage: int = 1):
    """ZeroPlan::make (parallel.cpp:20-34) -> (part_sizes, offsets)."""
    ps = (C.c_uint64 * max(dp_size, 1))()
    offs = (C.c_uint64 * (max(dp_size, 1) + 1))()
    _check(lib.mco_zero_plan(int(total_len), int(dp_size), int(stage), ps, offs))
    return [ps[i] for i in range(dp_size)], [offs[i] for i in range(dp_size + 1)]


def synth_fill(t, seed: int, role: int, tensor: int, step: int, cols: int = 0,
               scale_log2: int = 0, zero_log2: int = 0, rowcol: bool = False,
               stream=None) -> None:
    """Fill a CUDA tensor with the counter-based synthetic generator."""
    _dev(t, "synth")
    _check(lib.mco_synth_fill(t.data_ptr(), _dtype_code(t), t.numel(), int(seed), int(role),
                              int(tensor), int(step), int(cols), int(scale_log2),
                              int(zero_log2), int(rowcol), _stream(stream)))


def set_flat_variant(name: str) -> None:
    """Select the stored-state kernels' data-movement variant ("tma" default, "ldg")."""
    _check(lib.mco_set_flat_variant(name.encode()))


def flat_variant() -> str:
    return lib.mco_flat_variant().decode()


def host_release() -> None:
    """Free the device buffers the host-span calls keep between calls (lomo_step on host
    arrays with the clip keeps its resident gradient, mco_host_release)."""
    _check(lib.mco_host_release())


def launch_count() -> int:
    """Kernel launches issued by libmco in this process."""
    return int(lib.mco_launch_count())


def device_count() -> int:
    n = C.c_int()
    _check(lib.mco_device_count(C.byref(n)))
    return n.value
