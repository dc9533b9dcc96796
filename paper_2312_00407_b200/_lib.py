"""ctypes binding of the C-ABI (include/mco.h) -> _build/libmco.so.

The product path has no fallback: if the CUDA library is missing this module
raises at import, naming the build command.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("MCO_LIB_PATH") or os.path.join(HERE, "_build", "libmco.so")
HEADER = os.path.join(ROOT, "include", "mco.h")

MCO_OK, MCO_CONFIG, MCO_DATA, MCO_CONTRACT, MCO_PROTOCOL, MCO_IO, MCO_CUDA = 0, 2, 3, 4, 5, 6, 7
MCO_F32, MCO_BF16, MCO_F64, MCO_F32M64 = 0, 1, 2, 3


class mco_config(C.Structure):
    """include/mco.h mco_config == optim.hpp:20-35 OptimizerConfig."""

    _fields_ = [
        ("kind", C.c_int),
        ("lr", C.c_double),
        ("weight_decay", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("beta3", C.c_double),
        ("eps", C.c_double),
        ("has_clip_threshold", C.c_int),
        ("clip_threshold", C.c_double),
        ("adalomo_clip", C.c_double),
        ("sophia_rho", C.c_double),
        ("update_interval", C.c_int),
    ]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"paper_2312_00407_b200: CUDA library {LIB_PATH} is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'` or "
            "`make -C paper_2312_00407_b200/csrc`). There is no CPU fallback.")
    return C.CDLL(LIB_PATH)


lib = _load()

_p, _i, _u64, _i64, _d = C.c_void_p, C.c_int, C.c_uint64, C.c_int64, C.c_double
_cfgp = C.POINTER(mco_config)
_SIGS = {
    "mco_last_error": (C.c_char_p, []),
    "mco_version": (C.c_char_p, []),
    "mco_launch_count": (_u64, []),
    "mco_host_release": (_i, []),
    "mco_parse_kind": (_i, [C.c_char_p, C.POINTER(_i)]),
    "mco_kind_name": (C.c_char_p, [_i]),
    "mco_is_fused": (_i, [_i]),
    "mco_defaults_for": (_i, [_i, _cfgp]),
    "mco_validate": (_i, [_cfgp]),
    "mco_state_bytes": (_i, [_i, _u64, _i, _i, _i, _i, C.POINTER(_i), C.POINTER(_i64),
                             C.POINTER(_u64)]),
    "mco_flat_create": (_i, [_cfgp, _u64, _i, _i, C.POINTER(_p)]),
    "mco_flat_destroy": (_i, [_p]),
    "mco_flat_step": (_i, [_p, _p, _i, _u64, _p, _i, _u64, _d, _p]),
    "mco_flat_step_mixed": (_i, [_p, _p, _p, _i, _p, _u64, _d, _p]),
    "mco_flat_step_host": (_i, [_p, _p, _i, _u64, _p, _i, _u64, _d]),
    "mco_flat_get_steps": (_i, [_p, C.POINTER(_i64)]),
    "mco_flat_set_steps": (_i, [_p, _i64]),
    "mco_flat_graph_enable": (_i, [_p, _p]),
    "mco_flat_step_list": (_i, [_p, _i, C.POINTER(_p), _i, C.POINTER(_p), _i,
                                C.POINTER(_u64), _d, _p]),
    "mco_flat_graph_disable": (_i, [_p]),
    "mco_flat_state_bytes": (_i, [_p, C.POINTER(_u64)]),
    "mco_flat_config": (_i, [_p, _cfgp]),
    "mco_flat_num_buffers": (_i, [_p, C.POINTER(_i)]),
    "mco_flat_buffer": (_i, [_p, _i, C.POINTER(C.c_char_p), C.POINTER(_p), C.POINTER(_u64),
                             C.POINTER(_i)]),
    "mco_flat_step_peers": (_i, [_p, C.POINTER(_p), _i, C.POINTER(_p), _i, _i, _p, _u64, _u64,
                                 _d, _p]),
    "mco_sumsq_peers": (_i, [C.POINTER(_p), _i, _i, _u64, _u64, _p, _p]),
    "mco_lomo_apply_peers": (_i, [C.POINTER(_p), _i, C.POINTER(_p), _i, _i, _p, _u64, _u64, _d,
                                  _d, _p, _d, _p]),
    "mco_peer_alloc": (_i, [_u64, _i, C.POINTER(_p)]),
    "mco_peer_free": (_i, [_p]),
    "mco_peer_export": (_i, [_p, _p]),
    "mco_peer_import": (_i, [_p, _i, C.POINTER(_p)]),
    "mco_peer_close": (_i, [_p]),
    "mco_lomo_apply": (_i, [_p, _i, _p, _i, _u64, _d, _d, _p]),
    "mco_lomo_apply_clipped": (_i, [_p, _i, _p, _i, _u64, _d, _p, _d, _p]),
    "mco_lomo_apply_list": (_i, [_i, C.POINTER(_p), _i, C.POINTER(_p), _i, C.POINTER(_u64),
                                 _d, _d, _p, _d, _p]),
    "mco_sumsq": (_i, [_p, _i, _u64, _p, _i, _p]),
    "mco_lomo_apply_host": (_i, [_p, _i, _p, _i, _u64, _d, _d, _d]),
    "mco_adalomo_apply_all_host": (_i, [_p, _p, _i, _p, _i, _d]),
    "mco_adalomo_create": (_i, [_cfgp, _i, C.POINTER(_i), C.POINTER(_i64), _i, C.POINTER(_p)]),
    "mco_adalomo_destroy": (_i, [_p]),
    "mco_adalomo_apply": (_i, [_p, _i, _p, _i, _p, _i, _d, _p, _p]),
    "mco_adalomo_apply_all": (_i, [_p, _p, _i, _p, _i, _d, _p]),
    "mco_adalomo_apply_list": (_i, [_p, _i, _i, C.POINTER(_p), _i, C.POINTER(_p), _i, _d, _p,
                                    _p]),
    "mco_adalomo_state_bytes": (_i, [_p, C.POINTER(_u64)]),
    "mco_adalomo_set_shard": (_i, [_p, _i, _i64, _d]),
    "mco_adalomo_set_grad_clip": (_i, [_p, _i, _d]),
    "mco_adalomo_phase": (_i, [_p, _i, _p, _i, _p, _i, _d, _p]),
    "mco_adalomo_payload": (_i, [_p, _i, C.POINTER(_p), C.POINTER(_u64)]),
    "mco_adalomo_get_steps": (_i, [_p, _i, C.POINTER(_i64)]),
    "mco_adalomo_buffer": (_i, [_p, _i, _i, C.POINTER(_p), C.POINTER(_u64)]),
    "mco_zero_plan": (_i, [_u64, _i, _i, C.POINTER(_u64), C.POINTER(_u64)]),
    "mco_synth_fill": (_i, [_p, _i, _u64, _u64, C.c_uint32, C.c_uint32, C.c_uint32, _i64, _i,
                            _i, _i, _p]),
    "mco_sync": (_i, [_p]),
    "mco_device_count": (_i, [C.POINTER(_i)]),
    "mco_set_flat_variant": (_i, [C.c_char_p]),
    "mco_comm_unique_id": (_i, [_p]),
    "mco_comm_create": (_i, [_p, _i, _i, _i, C.POINTER(_p)]),
    "mco_comm_destroy": (_i, [_p]),
    "mco_comm_check": (_i, [_p]),
    "mco_comm_allreduce_sum": (_i, [_p, _p, _i, _u64, _p]),
    "mco_shard_step": (_i, [_p, _p, _p, _i, _p, _i, _u64, _d, _p]),
    "mco_shard_step_mixed": (_i, [_p, _p, _p, _p, _p, _i, _u64, _d, _p]),
    "mco_comm_create_timeout": (_i, [_p, _i, _i, _i, _d, C.POINTER(_p)]),
    "mco_comm_wait": (_i, [_p, _p]),
    "mco_comm_abort": (_i, [_p]),
    "mco_zb_create": (_i, [_p, _p, _u64, _u64, _i, _i, C.POINTER(_p)]),
    "mco_zb_destroy": (_i, [_p]),
    "mco_zb_info": (_i, [_p, C.POINTER(_u64), C.POINTER(_i), C.POINTER(_u64), C.POINTER(_p),
                         C.POINTER(_p)]),
    "mco_zb_piece": (_i, [_p, _i, _i, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64),
                          C.POINTER(_u64), C.POINTER(_u64)]),
    "mco_zb_load_master": (_i, [_p, _p, _i, _p]),
    "mco_zb_begin": (_i, [_p, _p, _d, _p]),
    "mco_zb_grad_buffer": (_i, [_p, _i, C.POINTER(_p), C.POINTER(_u64), _p]),
    "mco_zb_grad_ready": (_i, [_p, _i, _p, _p]),
    "mco_zb_end": (_i, [_p, _p]),
    "mco_zb_step": (_i, [_p, _p, _p, _d, _p]),
    "mco_zb_gathered": (_i, [_p, _i, C.POINTER(_p), _p]),
    "mco_zb_step_local": (_i, [_p, _p, _p, _d, _p]),
    "mco_zb_plan": (_i, [_u64, _i, _u64, _i, _i, C.POINTER(_u64), C.POINTER(_i),
                         C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "mco_flat_variant": (C.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def header_symbols() -> list[str]:
    """Every function the C header declares (the exported-symbol contract)."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mco_[a-z0-9_]+)\s*\(", text)))
