"""CPU-side checks of the C ABI boundary: the in-tree library builds for
sm_100a, loads, exports every entry point include/rimdp_b200.h declares, and
fails loudly (no fallback) when no device is visible."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2401_04068_b200 import build, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rimdp_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(rimdp_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for required in ("rimdp_model_create", "rimdp_model_destroy", "rimdp_solve", "rimdp_bellman_step",
                     "rimdp_column_values", "rimdp_last_error", "rimdp_model_generate"):
        assert required in fns


def test_library_exports_every_declared_symbol(engine_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", engine.library_path()], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (rimdp_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", engine.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_abi_version_and_error_path_without_device(engine_lib):
    assert engine_lib.rimdp_abi_version() == 4
    if engine.device_count() > 0:
        pytest.skip("a device is visible")
    with pytest.raises(engine.EngineError) as ei:
        engine.DeviceModel.from_csc([0, 1], [0, 1], [0], np.array([1.0]), np.array([1.0]))
    assert ei.value.status == engine.ERR_NO_DEVICE


def test_invalid_arguments_rejected_before_device_work(engine_lib):
    desc = engine.ModelDesc()
    h = C.c_void_p()
    assert engine_lib.rimdp_model_create(None, C.byref(h)) == engine.ERR_INVALID_ARGUMENT
    sp = np.array([0, 1], np.int32)
    cp = np.array([0, 2], np.int64)  # colptr end != nnz
    rv = np.zeros(1, np.int32)
    lo = np.ones(1)
    desc = engine.ModelDesc(0, 0, 1, 1, 1, sp.ctypes.data, cp.ctypes.data, rv.ctypes.data, lo.ctypes.data,
                            lo.ctypes.data)
    assert engine_lib.rimdp_model_create(C.byref(desc), C.byref(h)) == engine.ERR_INVALID_ARGUMENT
    assert b"colptr" in engine_lib.rimdp_last_error()


def test_build_is_up_to_date_after_build():
    build.build()
    assert build.up_to_date()
