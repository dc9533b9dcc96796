"""C-ABI boundary checks that need no GPU: the library loads, exports exactly the
symbols include/mco.h declares, and its host-side logic behaves like the reference."""
import ctypes as C
import subprocess

import pytest

from paper_2312_00407_b200 import _lib, optim


def test_library_exports_every_header_symbol():
    declared = _lib.header_symbols()
    assert len(declared) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    extra = sorted(s for s in exported if not s.startswith("mco_"))
    assert not extra, extra  # nothing but the C-ABI leaks out
    for s in declared:
        assert getattr(_lib.lib, s) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_89"):
        assert other not in out


def test_fused_kind_rejected_by_flat_optimizer():
    # optim.cpp:93-96: checked on the host before any device work
    for k in (optim.Kind.LOMO, optim.Kind.ADALOMO):
        with pytest.raises(optim.ContractError, match="is a fused optimizer"):
            optim.FlatOptimizer(optim.OptimizerConfig.defaults_for(k), 10)


def test_zero_plan_errors():
    with pytest.raises(optim.ConfigError, match="dp_size must be >= 1"):
        optim.zero_plan(10, 0)
    with pytest.raises(optim.ConfigError, match="stage must be in 0..3"):
        optim.zero_plan(10, 2, stage=4)


def test_config_struct_layout_matches_header():
    # mco_config is passed by pointer across the boundary; pin its size / offsets
    assert C.sizeof(_lib.mco_config) == 96
    assert _lib.mco_config.update_interval.offset == 88


def test_no_gpu_reports_zero_devices_or_real_count():
    assert optim.device_count() >= 0


def test_flat_variant_knob_host_side():
    from paper_2312_00407_b200 import optim

    prev = optim.flat_variant()
    with pytest.raises(optim.ConfigError, match="unknown flat-kernel variant 'nope'"):
        optim.set_flat_variant("nope")
    assert optim.flat_variant() == prev
    optim.set_flat_variant("ldg")
    assert optim.flat_variant() == "ldg"
    optim.set_flat_variant(prev)


def test_null_handles_are_contract_errors():
    """Every entry point taking a handle (mco_flat / mco_adalomo / mco_comm) returns
    MCO_CONTRACT with a message for a NULL handle, before touching the device."""
    import re

    header = open(_lib.HEADER_PATH).read() if hasattr(_lib, "HEADER_PATH") else None
    if header is None:
        import os

        header = open(os.path.join(os.path.dirname(os.path.dirname(_lib.__file__)), "include",
                                   "mco.h")).read()
    decls = re.findall(r"mco_status (mco_\w+)\(([^;]*?)\);", header, re.S)
    checked = 0
    for name, args in decls:
        first = args.split(",")[0]
        if not re.search(r"mco_(flat|adalomo|comm)\s*\*", first) or name.endswith("destroy"):
            continue
        fn = getattr(_lib.lib, name)
        argv = []
        for t in fn.argtypes:
            if t in (C.c_double, C.c_float):
                argv.append(0.0)
            elif t in (C.c_int, C.c_int64, C.c_uint64, C.c_uint32):
                argv.append(0)
            else:
                argv.append(None)
        assert fn(*argv) == _lib.MCO_CONTRACT, name
        assert "null handle" in _lib.lib.mco_last_error().decode(), name
        checked += 1
    assert checked >= 25


def test_null_data_pointers_are_contract_errors():
    """n > 0 elements behind a NULL pointer is refused on the host (it would fault on
    the device and poison the context)."""
    L = _lib.lib
    assert L.mco_lomo_apply(None, _lib.MCO_F32, None, _lib.MCO_F32, 8, 1e-3, 1.0,
                            None) == _lib.MCO_CONTRACT
    assert "null data pointer" in L.mco_last_error().decode()
    assert L.mco_lomo_apply_host(None, _lib.MCO_F32, None, _lib.MCO_F32, 8, 1e-3, 1.0,
                                 -1.0) == _lib.MCO_CONTRACT
    assert L.mco_sumsq(None, _lib.MCO_F32, 8, None, 0, None) == _lib.MCO_CONTRACT
