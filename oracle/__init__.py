"""TEST INFRASTRUCTURE ONLY — the CPU checkers for the B200 engine.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline — never as the product path.

Two checkers, same Python surface:

* ``ref``  — the reference itself (``/root/reference/proj/include`` headers,
  compiled in place by ``oracle/Makefile`` into ``oracle/_ref/librimdp_ref.so``).
* ``port`` — ``oracle/port/rimdp_port.c``, a plain-C restatement of the hot
  path (omax.hpp / bellman.hpp / solver.hpp), pinned against ``ref`` and the
  golden fixtures in ``tests/golden``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "librimdp_ref.so")
PORT_SO = os.path.join(HERE, "_port", "librimdp_port.so")
REFERENCE_ROOT = os.environ.get("RIMDP_REFERENCE", "/root/reference")

# property kinds (reference property.hpp:14-59, variant order)
FINITE_REACH, INFINITE_REACH, FINITE_REACH_AVOID, INFINITE_REACH_AVOID, FINITE_REWARD, INFINITE_REWARD = range(6)
STATUS = {0: "ok", 1: "ModelError", 2: "NonConvergence", 3: "PropertyStateOutOfRange",
          4: "InvalidProperty", 5: "InvalidPolicyAction", 9: "Error"}


def build(ref: bool = True, port: bool = True, quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle).  _ref only when the reference is present."""
    targets = []
    if port:
        targets.append("port")
    if ref and os.path.isdir(os.path.join(REFERENCE_ROOT, "proj", "include")):
        targets.append("ref")
    if targets:
        subprocess.run(["make", "-s", "-C", HERE, f"REF={REFERENCE_ROOT}", *targets], check=True,
                       stdout=subprocess.DEVNULL if quiet else None)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


class Spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("reach", C.POINTER(C.c_int)), ("nreach", C.c_int),
                ("avoid", C.POINTER(C.c_int)), ("navoid", C.c_int), ("rewards", C.c_void_p),
                ("discount", C.c_double), ("horizon", C.c_longlong), ("eps", C.c_double),
                ("pessimistic", C.c_int), ("maximize", C.c_int), ("workers", C.c_uint),
                ("max_iterations", C.c_longlong)]


class Err(C.Structure):
    _fields_ = [("msg", C.c_char * 512), ("iterations", C.c_longlong), ("residual", C.c_double),
                ("violation_kind", C.c_int), ("violation_column", C.c_longlong)]


class OracleError(RuntimeError):
    def __init__(self, status: int, err: Err):
        self.kind = STATUS.get(status, "Error")
        self.status = status
        self.message = err.msg.decode(errors="replace")
        self.iterations = int(err.iterations)
        self.residual = float(err.residual)
        self.violation_kind = int(err.violation_kind)
        super().__init__(f"{self.kind}: {self.message}")


@dataclass
class Problem:
    """Plain description of a solve, shared by every checker and the engine tests."""
    kind: int
    reach: list = field(default_factory=list)
    avoid: list = field(default_factory=list)
    rewards: np.ndarray | None = None
    discount: float = 0.0
    horizon: int = 0
    eps: float = 0.0
    pessimistic: bool = True
    maximize: bool = True
    max_iterations: int = 1_000_000


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run oracle.build())")
        self.lib = C.CDLL(path)
        self.prefix = prefix

    def fn(self, name, dtype):
        suffix = "_f64" if np.dtype(dtype) == np.float64 else "_f32"
        return getattr(self.lib, f"{self.prefix}{name}{suffix}")


_libs: dict = {}


def _lib(which: str) -> _Lib:
    if which not in _libs:
        _libs[which] = _Lib(REF_SO, "ref_") if which == "ref" else _Lib(PORT_SO, "port_")
    return _libs[which]


def _spec(p: Problem, n: int, dtype, workers: int, keep: list) -> Spec:
    reach = np.ascontiguousarray(p.reach, dtype=np.int32)
    avoid = np.ascontiguousarray(p.avoid, dtype=np.int32)
    keep += [reach, avoid]
    rew = None
    if p.rewards is not None:
        rew = np.ascontiguousarray(p.rewards, dtype=dtype)
        keep.append(rew)
    return Spec(p.kind, _ptr(reach, C.c_int), len(reach), _ptr(avoid, C.c_int), len(avoid),
                rew.ctypes.data if rew is not None else None, float(p.discount), int(p.horizon),
                float(p.eps), int(p.pessimistic), int(p.maximize), int(workers), int(p.max_iterations))


class Model:
    """A model held by one checker ("ref" or "port"), built from CSC arrays."""

    def __init__(self, which: str, handle, dtype):
        self.which, self.h, self.dtype = which, handle, np.dtype(dtype)
        self.L = _lib(which)

    def __del__(self):
        try:
            if self.h:
                self.L.lib[f"{self.L.prefix}model_free"](self.h)
        except Exception:
            pass

    @classmethod
    def from_arrays(cls, which, stateptr, colptr, rowval, lower, upper, checked=True):
        dtype = np.asarray(lower).dtype
        L = _lib(which)
        sp = np.ascontiguousarray(stateptr, np.int32)
        cp = np.ascontiguousarray(colptr, np.int32) if which == "ref" else np.ascontiguousarray(colptr, np.int64)
        rv = np.ascontiguousarray(rowval, np.int32)
        lo = np.ascontiguousarray(lower, dtype)
        up = np.ascontiguousarray(upper, dtype)
        h = C.c_void_p()
        err = Err()
        f = L.fn("model_from_arrays", dtype)
        ct = C.c_double if dtype == np.float64 else C.c_float
        cpt = C.c_int if which == "ref" else C.c_longlong
        st = f(len(sp) - 1, len(cp) - 1, _ptr(sp, C.c_int), _ptr(cp, cpt), _ptr(rv, C.c_int),
               _ptr(lo, ct), _ptr(up, ct), int(checked), C.byref(h), C.byref(err))
        if st:
            raise OracleError(st, err)
        return cls(which, h, dtype)

    @classmethod
    def random(cls, states, actions, density, scale, seed, point=False, dtype=np.float64):
        """The reference's own generator (random_model.hpp:42-161); ref only."""
        L = _lib("ref")
        h = C.c_void_p()
        err = Err()
        st = L.fn("model_random", dtype)(int(states), int(actions), C.c_double(density), C.c_double(scale),
                                         C.c_ulonglong(seed), int(point), C.byref(h), C.byref(err))
        if st:
            raise OracleError(st, err)
        return cls("ref", h, dtype)

    @classmethod
    def generate(cls, states, actions, *, law=0, support=64, alpha=1.5, kmax=4096, lower_scale=None,
                 upper_scale=None, seed=1, dtype=np.float64):
        """A counter-generator workload (configs 4-5, csrc/generator.cuh host build) built through the
        reference's checked constructors; ref only.  Scales default as engine.gen_config."""
        if law == 0:
            k = min(support, states)
            lower_scale = 1.0 / k if lower_scale is None else lower_scale
            upper_scale = 1.0 - 1.0 / k if upper_scale is None else upper_scale
        else:
            lower_scale = 0.5 if lower_scale is None else lower_scale
            upper_scale = 3.0 if upper_scale is None else upper_scale
        L = _lib("ref")
        h = C.c_void_p()
        err = Err()
        st = L.fn("model_generate", dtype)(int(states), int(actions), int(law), int(support), C.c_double(alpha),
                                           int(kmax), C.c_double(lower_scale), C.c_double(upper_scale),
                                           C.c_ulonglong(seed), C.byref(h), C.byref(err))
        if st:
            raise OracleError(st, err)
        return cls("ref", h, dtype)

    @classmethod
    def read_native(cls, path, dtype=np.float64):
        """io::read_native_model (io/native.hpp:457-561) of the reference; ref only."""
        L = _lib("ref")
        h = C.c_void_p()
        err = Err()
        st = L.fn("read_native", dtype)(os.fsencode(path), C.byref(h), C.byref(err))
        if st:
            raise OracleError(st, err)
        return cls("ref", h, dtype)

    def write_native(self, path, json_debug=False):
        """io::write_native_model (io/native.hpp:424-455); ref models only."""
        err = Err()
        st = self.L.fn("write_native", self.dtype)(self.h, os.fsencode(path), int(json_debug), C.byref(err))
        if st:
            raise OracleError(st, err)

    def labels(self):
        """The model's action labels (IntervalMDP::actions, imdp.hpp:108); ref models only."""
        f = self.L.fn("model_labels", self.dtype)
        f.restype = C.c_longlong
        nb = f(self.h, None)
        buf = C.create_string_buffer(max(int(nb), 1))
        f(self.h, buf)
        return [x.decode() for x in buf.raw[:nb].split(b"\0")[:-1]]

    def sizes(self):
        n, nc, nnz = C.c_int(), C.c_int(), C.c_longlong()
        self.L.fn("model_sizes", self.dtype)(self.h, C.byref(n), C.byref(nc), C.byref(nnz))
        return n.value, nc.value, nnz.value

    def export(self):
        """(stateptr int32, colptr int64, rowval int32, lower, upper) — ref models only."""
        n, nc, nnz = self.sizes()
        sp = np.empty(n + 1, np.int32)
        cp = np.empty(nc + 1, np.int32)
        rv = np.empty(nnz, np.int32)
        lo = np.empty(nnz, self.dtype)
        up = np.empty(nnz, self.dtype)
        ct = C.c_double if self.dtype == np.float64 else C.c_float
        self.L.fn("model_export", self.dtype)(self.h, _ptr(sp, C.c_int), _ptr(cp, C.c_int), _ptr(rv, C.c_int),
                                              _ptr(lo, ct), _ptr(up, ct))
        return sp, cp.astype(np.int64), rv, lo, up

    def solve(self, p: Problem, synthesize=False, workers=0, trace_iters=0):
        n, _, _ = self.sizes()
        keep: list = []
        spec = _spec(p, n, self.dtype, workers, keep)
        ct = C.c_double if self.dtype == np.float64 else C.c_float
        v = np.empty(n, self.dtype)
        r = np.empty(n, self.dtype)
        it = C.c_longlong()
        finite = p.kind in (FINITE_REACH, FINITE_REACH_AVOID, FINITE_REWARD)
        pol = None
        if synthesize:
            pol = np.full(n * (p.horizon if finite else 1), -7, np.int32)
        trace = np.zeros((trace_iters, n), self.dtype) if trace_iters else None
        err = Err()
        st = self.L.fn("solve", self.dtype)(self.h, C.byref(spec), int(synthesize), _ptr(v, ct), _ptr(r, ct),
                                            C.byref(it), _ptr(pol, C.c_int), _ptr(trace, ct),
                                            C.c_longlong(trace_iters), C.byref(err))
        if st:
            raise OracleError(st, err)
        out = {"values": v, "residual": r, "iterations": it.value}
        if synthesize:
            out["policy"] = pol.reshape(n, -1) if finite else pol
        if trace is not None:
            out["trace"] = trace
        return out

    def verify_policy(self, p: Problem, policy_cols, workers=0):
        n, _, _ = self.sizes()
        keep: list = []
        spec = _spec(p, n, self.dtype, workers, keep)
        pol = np.ascontiguousarray(policy_cols, np.int32)
        td = pol.ndim == 2
        ct = C.c_double if self.dtype == np.float64 else C.c_float
        v = np.empty(n, self.dtype)
        r = np.empty(n, self.dtype)
        it = C.c_longlong()
        err = Err()
        st = self.L.fn("verify_policy", self.dtype)(self.h, C.byref(spec), _ptr(pol, C.c_int), int(td),
                                                    C.c_longlong(pol.shape[1] if td else 0), _ptr(v, ct),
                                                    _ptr(r, ct), C.byref(it), C.byref(err))
        if st:
            raise OracleError(st, err)
        return {"values": v, "residual": r, "iterations": it.value}

    def bellman_step(self, values, pessimistic, maximize, frozen=None, workers=0):
        n, _, _ = self.sizes()
        ct = C.c_double if self.dtype == np.float64 else C.c_float
        v = np.ascontiguousarray(values, self.dtype)
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.uint8)
        ov = np.empty(n, self.dtype)
        oc = np.empty(n, np.int32)
        err = Err()
        st = self.L.fn("bellman_step", self.dtype)(self.h, _ptr(v, ct), int(pessimistic), int(maximize),
                                                   _ptr(fz, C.c_ubyte), int(workers), _ptr(ov, ct),
                                                   _ptr(oc, C.c_int), C.byref(err))
        if st:
            raise OracleError(st, err)
        return ov, oc


def generate_nnz(states, actions, *, law=0, support=64, alpha=1.5, kmax=4096, seed=1) -> int:
    """Transitions of a counter-generator workload (column lengths only, any size)."""
    f = _lib("ref").lib.ref_generate_nnz
    f.restype = C.c_longlong
    return int(f(int(states), int(actions), int(law), int(support), C.c_double(alpha), int(kmax),
                 C.c_ulonglong(seed)))


def robust_expectation(which, rows, lower, upper, values, pessimistic, with_p=False):
    """Column-level entry point (omax.hpp:182-189)."""
    dtype = np.asarray(lower).dtype
    L = _lib(which)
    ct = C.c_double if dtype == np.float64 else C.c_float
    rows = np.ascontiguousarray(rows, np.int32)
    lo = np.ascontiguousarray(lower, dtype)
    up = np.ascontiguousarray(upper, dtype)
    vals = np.ascontiguousarray(values, dtype)
    out = (C.c_double if dtype == np.float64 else C.c_float)()
    p = np.empty(len(rows), dtype) if with_p else None
    err = Err()
    st = L.fn("robust_expectation", dtype)(len(rows), _ptr(rows, C.c_int), _ptr(lo, ct), _ptr(up, ct),
                                           _ptr(vals, ct), int(pessimistic), C.byref(out), _ptr(p, ct),
                                           C.byref(err))
    if st:
        raise OracleError(st, err)
    return (out.value, p) if with_p else out.value


def lp_expectation(lower, upper, values, minimize):
    """The reference test-suite's break-point LP (tests/oracle.hpp:28-80)."""
    L = _lib("ref")
    f = L.lib.ref_lp_expectation_f64
    f.restype = C.c_double
    lo = np.ascontiguousarray(lower, np.float64)
    up = np.ascontiguousarray(upper, np.float64)
    v = np.ascontiguousarray(values, np.float64)
    return f(len(lo), _ptr(lo, C.c_double), _ptr(up, C.c_double), _ptr(v, C.c_double), int(minimize))


def test_columns(seed, count, nmin=1, nmod=10, scale=0.3, with_values=True):
    """The reference tests' random feasible columns (tests/oracle.hpp:187-217)."""
    L = _lib("ref")
    f = L.lib.ref_test_columns_f64
    f.restype = C.c_longlong
    cap = count * (nmin + nmod)
    lens = np.empty(count, np.int32)
    lo = np.empty(cap)
    up = np.empty(cap)
    vals = np.empty(cap)
    tot = f(C.c_ulonglong(seed), count, nmin, nmod, C.c_double(scale), int(with_values), _ptr(lens, C.c_int),
            _ptr(lo, C.c_double), _ptr(up, C.c_double), _ptr(vals, C.c_double), C.c_longlong(cap))
    return lens, lo[:tot], up[:tot], vals[:tot]
