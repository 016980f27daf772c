"""In-tree build of the sm_100a engine library (no JIT cache, no pip install).

``build()`` compiles ``csrc/*.cu`` with nvcc for ``sm_100a`` into
``paper_2401_04068_b200/lib/librimdp_b200.so`` — the file that travels to
the GPU box with the gpurun snapshot and that the ctypes binding loads.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "librimdp_b200.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
              "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 engine cannot be built")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def host_sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")))


def deps() -> list[str]:
    return (sources() + host_sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) +
            sorted(glob.glob(os.path.join(INCLUDE, "rimdp_b200*.h"))))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Compile every .cu under csrc into one shared library for sm_100a
    (`out` / `defines`: an alternative build for kernel experiments)."""
    if out is None and not force and up_to_date():
        return LIB
    lib_path = out or LIB
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(LIBDIR, os.path.basename(src) + ".o")
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC, "-c", src,
               "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    for src in host_sources():
        obj = os.path.join(LIBDIR, os.path.basename(src) + ".o")
        # plain mul/add rounding, like the reference build (no FMA contraction)
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-ffp-contract=off", "-I", INCLUDE, "-c", src,
               "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib_path + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", *objs, "-o", tmp, "-lcudart"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib_path)
    for o in objs:
        os.remove(o)
    return lib_path


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "dropin_parity.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_parity")
REFERENCE_INCLUDE = os.path.join(os.environ.get("RIMDP_REFERENCE", "/root/reference"), "proj", "include")


def build_cpp_tests(force: bool = False) -> str | None:
    """Compile the C++ drop-in parity program (tests/cpp/dropin_parity.cpp):
    include/rimdp_b200/dropin.hpp over the engine library, checked against the
    reference's own headers compiled in as the oracle.  Needs the reference
    headers (present in the build container, absent on the GPU box, where the
    prebuilt binary travels with the snapshot); returns None without them."""
    if not os.path.isdir(REFERENCE_INCLUDE):
        return None
    deps_ = [CPP_TEST_SRC, os.path.join(INCLUDE, "rimdp_b200", "dropin.hpp"), os.path.join(INCLUDE, "rimdp_b200.h")]
    if (not force and os.path.exists(CPP_TEST_BIN) and
            all(os.path.getmtime(d) <= os.path.getmtime(CPP_TEST_BIN) for d in deps_)):
        return CPP_TEST_BIN
    os.makedirs(os.path.dirname(CPP_TEST_BIN), exist_ok=True)
    stubs = os.path.join(ROOT, "oracle", "stubs")  # Boost stub: Rational is never instantiated
    # nlohmann/json 3.11.3 for the reference's io/native.hpp (container parity cases)
    import sysconfig
    json_inc = os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty", "nlohmann")
    cmd = ["g++", "-std=gnu++20", "-O2", "-Wall", "-Wextra", "-Wno-unused-parameter", "-ffp-contract=off",
           "-I", stubs, "-I", REFERENCE_INCLUDE, "-I", INCLUDE, "-I", json_inc, CPP_TEST_SRC, "-o", CPP_TEST_BIN,
           "-L", LIBDIR, "-lrimdp_b200", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,$ORIGIN/../../../paper_2401_04068_b200/lib",
           "-pthread"]
    subprocess.run(cmd, check=True)
    return CPP_TEST_BIN


if __name__ == "__main__":
    print(build(force=True, verbose=True))
