"""B200-native robust value iteration for interval MDPs.

The drop-in host API for C++ callers is ``include/rimdp_b200/dropin.hpp`` over the C
ABI ``include/rimdp_b200.h``; this package holds the CUDA sources
(``csrc/``), the in-tree build, the ctypes binding and the Python-side
problem helpers used by tests, the benchmark and the sharded driver.
"""
from . import build, engine  # noqa: F401
from .engine import DeviceModel, EngineError  # noqa: F401

__all__ = ["build", "engine", "DeviceModel", "EngineError"]
