"""The C++ drop-in layer (include/rimdp_b200/dropin.hpp): the reference's own
entry points and the engine's, called on the same Problem objects in one C++
process (tests/cpp/dropin_parity.cpp)."""
import os
import subprocess

import pytest

from paper_2401_04068_b200 import build, engine


def _binary():
    path = build.build_cpp_tests()  # rebuilt here when the reference headers are present
    if path is None:
        path = build.CPP_TEST_BIN if os.path.exists(build.CPP_TEST_BIN) else None
    if path is None:
        pytest.skip("dropin_parity not built (needs the reference headers at build time)")
    return path


def test_dropin_header_compiles_and_fails_loudly_without_device(engine_lib):
    if engine.device_count() > 0:
        pytest.skip("a device is visible: the no-device path is not reachable")
    r = subprocess.run([_binary(), "--no-device"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_dropin_parity_against_reference_entry_points(engine_lib):
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=1200)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failures" in r.stdout
