"""ctypes binding of the C ABI in include/rimdp_b200.h.

This is plumbing for tests, bench.py and the sharded driver; the drop-in
host API for C++ callers is include/rimdp_b200/dropin.hpp.  The library is loaded from
the package tree (``lib/librimdp_b200.so``); there is no CPU fallback — if
the library is missing, building or loading raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import build as _build

RIMDP_F64, RIMDP_F32 = 0, 1
(OK, ERR_INVALID_ARGUMENT, ERR_INFEASIBLE_COLUMN, ERR_NON_CONVERGENCE, ERR_CUDA, ERR_OOM, ERR_NO_DEVICE, ERR_INTERNAL,
 ERR_MISSING_FILE, ERR_SCHEMA, ERR_INVALID_MODEL) = range(11)
# rimdp::ViolationKind (reference errors.hpp:18-27)
VIOLATION_KINDS = ("ShapeMismatch", "EntryOutOfRange", "BoundOrderViolation", "InfeasibleColumn",
                   "DestinationCountMismatch", "DuplicateActionLabel", "EmptyActionSet", "StructuralError")


class EngineError(RuntimeError):
    """A non-zero rimdp_status with the thread's rimdp_last_error() text."""

    def __init__(self, status: int, message: str, info: "ErrorInfo"):
        self.status = status
        self.message = message
        self.iterations = int(info.iterations)
        self.residual = float(info.residual)
        self.column = int(info.column)
        self.violation_kind = int(info.violation_kind)
        self.row = int(info.row)
        super().__init__(f"rimdp status {status}: {message}")


class ErrorInfo(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_int64), ("residual", C.c_double),
                ("column", C.c_int64), ("infeasible_kind", C.c_int32), ("infeasible_sum", C.c_double),
                ("violation_kind", C.c_int32), ("row", C.c_int64)]


class ModelDesc(C.Structure):
    _fields_ = [("dtype", C.c_int), ("device", C.c_int32), ("num_states", C.c_int32), ("num_cols", C.c_int32),
                ("nnz", C.c_int64), ("stateptr", C.c_void_p), ("colptr", C.c_void_p), ("rowval", C.c_void_p),
                ("lower", C.c_void_p), ("upper", C.c_void_p)]


class GenConfig(C.Structure):
    _fields_ = [("dtype", C.c_int), ("device", C.c_int32), ("num_states", C.c_int32), ("actions", C.c_int32),
                ("law", C.c_int32), ("support", C.c_int32), ("alpha", C.c_double), ("kmax", C.c_int32),
                ("lower_scale", C.c_double), ("upper_scale", C.c_double), ("seed", C.c_uint64),
                ("state_begin", C.c_int32), ("state_end", C.c_int32)]


class ModelInfo(C.Structure):
    _fields_ = [("dtype", C.c_int), ("device", C.c_int32), ("num_states", C.c_int32), ("num_cols", C.c_int32),
                ("nnz", C.c_int64), ("state_begin", C.c_int32), ("state_end", C.c_int32),
                ("max_column_length", C.c_int32), ("num_infeasible_columns", C.c_int32),
                ("device_bytes", C.c_int64), ("short_columns", C.c_int32), ("mid_columns", C.c_int32),
                ("long_columns", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("pessimistic", C.c_int32), ("maximize", C.c_int32), ("finite", C.c_int32), ("horizon", C.c_int64),
                ("eps", C.c_double), ("max_iterations", C.c_int64), ("initial", C.c_void_p), ("frozen", C.c_void_p),
                ("rewards", C.c_void_p), ("discount", C.c_double), ("forced", C.c_void_p),
                ("forced_time_dependent", C.c_int32), ("external_stop", C.c_int32)]


ITER_CB = C.CFUNCTYPE(None, C.c_int64, C.c_void_p, C.c_void_p)


class Outputs(C.Structure):
    _fields_ = [("values", C.c_void_p), ("residual", C.c_void_p), ("iterations", C.POINTER(C.c_int64)),
                ("chosen", C.c_void_p), ("record_all_steps", C.c_int32), ("on_iteration", ITER_CB),
                ("user", C.c_void_p)]


_lib = None
_lock = threading.Lock()

_VP, _I32, _I64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_SIGNATURES = {
    # every entry point of include/rimdp_b200.h and rimdp_b200_workloads.h
    "rimdp_last_error": ([], C.c_char_p),
    "rimdp_last_error_info": ([_VP], C.c_int),
    "rimdp_abi_version": ([], C.c_int),
    "rimdp_device_count": ([_VP], C.c_int),
    "rimdp_model_create": ([_VP, _VP], C.c_int),
    "rimdp_model_destroy": ([_VP], C.c_int),
    "rimdp_model_create_shard": ([_VP, _I32, _I32, _VP], C.c_int),
    "rimdp_model_set_value_capacity": ([_VP, _I64], C.c_int),
    "rimdp_solve_residual_slots": ([_VP, _VP], C.c_int),
    "rimdp_solve_stop_test": ([_VP], C.c_int),
    "rimdp_model_generate": ([_VP, _VP], C.c_int),
    "rimdp_model_read_columns": ([_VP, _I32, _I32, _VP, _VP, _VP, _VP], C.c_int),
    "rimdp_model_info_get": ([_VP, _VP], C.c_int),
    "rimdp_model_stream": ([_VP, _VP], C.c_int),
    "rimdp_solve": ([_VP, _VP, _VP], C.c_int),
    "rimdp_solve_begin": ([_VP, _VP], C.c_int),
    "rimdp_solve_advance": ([_VP, _I64], C.c_int),
    "rimdp_solve_poll": ([_VP, _VP, _VP, _VP], C.c_int),
    "rimdp_solve_finish": ([_VP, _VP], C.c_int),
    "rimdp_solve_value_buffers": ([_VP, _VP, _VP], C.c_int),
    "rimdp_profile_enable": ([_VP, _I32], C.c_int),
    "rimdp_profile_read": ([_VP, _VP, _VP, _VP, _VP, _VP], C.c_int),
    "rimdp_bellman_step": ([_VP, _VP, _I32, _I32, _VP, _VP, _VP, _VP], C.c_int),
    "rimdp_column_values": ([_VP, _VP, _I32, _VP], C.c_int),
    "rimdp_generate_host": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP], C.c_int),
    "rimdp_native_read": ([C.c_char_p, _I32, _VP, _VP], C.c_int),
    "rimdp_native_take": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP], C.c_int),
    "rimdp_native_free": ([_VP], None),
    "rimdp_native_write": ([C.c_char_p, _I32, _I32, _I32, _VP, _VP, _VP, _VP, _VP, C.c_char_p, _I32], C.c_int),
    "rimdp_exchange_export": ([_VP, _VP], C.c_int),
    "rimdp_exchange_connect": ([_VP, _I32, _I32, _VP], C.c_int),
    "rimdp_exchange_connect_local": ([_VP, _I32], C.c_int),
    "rimdp_multi_create": ([_VP, _I32, _VP, _VP], C.c_int),
    "rimdp_multi_solve": ([_VP, _VP, _VP], C.c_int),
    "rimdp_multi_info": ([_VP, _VP, _VP, _VP], C.c_int),
    "rimdp_multi_destroy": ([_VP], C.c_int),
    "rimdp_random_imdp": ([_I32, _I32, _D, _D, C.c_uint64, _I32, _I32, _VP, _VP], C.c_int),
    "rimdp_random_imdp_take": ([_VP, _VP, _VP, _VP, _VP, _VP], C.c_int),
}


def _declare(lib) -> None:
    """Full prototypes: pointers must never be narrowed to C int."""
    for name, (args, res) in _SIGNATURES.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load the engine library, building it in-tree first if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("RIMDP_B200_LIB", _build.LIB)  # experiments: an alternative in-tree build
            if not os.path.exists(path):
                if not build_if_missing or path != _build.LIB:
                    raise FileNotFoundError(f"engine library not built: {path}")
                _build.build()
            lib = C.CDLL(path)
            _declare(lib)
            _lib = lib
    return _lib


def _check(status: int) -> None:
    if status != OK:
        lib = load()
        info = ErrorInfo()
        lib.rimdp_last_error_info(C.byref(info))
        raise EngineError(status, lib.rimdp_last_error().decode(errors="replace"), info)


def device_count() -> int:
    c = C.c_int()
    _check(load().rimdp_device_count(C.byref(c)))
    return c.value


class RandomSizes(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("num_cols", C.c_int32), ("nnz", C.c_int64)]


def random_imdp(states, actions, density, scale=0.2, seed=1, point=False, dtype=np.float64):
    """The reference generator's model (random_model.hpp:42-161) as CSC arrays:
    (stateptr int32, colptr int64, rowval int32, lower, upper)."""
    lib = load()
    sz = RandomSizes()
    h = C.c_void_p()
    st = lib.rimdp_random_imdp(C.c_int32(states), C.c_int32(actions), C.c_double(density), C.c_double(scale),
                               C.c_uint64(seed), C.c_int32(int(point)), C.c_int32(_dt(dtype)), C.byref(sz),
                               C.byref(h))
    if st:
        raise ValueError("rimdp_random_imdp: invalid configuration")
    sp = np.empty(sz.num_states + 1, np.int32)
    cp = np.empty(sz.num_cols + 1, np.int64)
    rv = np.empty(sz.nnz, np.int32)
    lo = np.empty(sz.nnz, dtype)
    up = np.empty(sz.nnz, dtype)
    lib.rimdp_random_imdp_take(h, _p(sp), _p(cp), _p(rv), _p(lo), _p(up))
    return sp, cp, rv, lo, up


def gen_config(num_states, actions, *, law=0, support=64, alpha=1.5, kmax=4096, lower_scale=None,
               upper_scale=None, seed=1, dtype=np.float64, device=0, state_begin=0, state_end=0) -> GenConfig:
    """A counter-based generator configuration (csrc/generator.cuh).

    law 0: `support` stratified rows per column, the reference generator's value law
    (lower = u/k, upper = min(lower + v (1 - 1/k), 1)) by default;
    law 1: power-law lengths k ~ k^-alpha on [1, kmax], lower = u * 0.5 / k,
    upper = min(lower + v * 3 / k, 1) by default."""
    if law == 0:
        k = min(support, num_states)
        lower_scale = 1.0 / k if lower_scale is None else lower_scale
        upper_scale = 1.0 - 1.0 / k if upper_scale is None else upper_scale
    else:
        lower_scale = 0.5 if lower_scale is None else lower_scale
        upper_scale = 3.0 if upper_scale is None else upper_scale
    return GenConfig(_dt(dtype), device, num_states, actions, law, support, alpha, kmax, lower_scale, upper_scale,
                     seed, state_begin, state_end)


def generate_host(cfg: GenConfig):
    """The generator on the host (bit-identical to rimdp_model_generate):
    (stateptr int32, colptr int64, rowval int32, lower, upper) of the configured shard."""
    lib = load()
    nc, nnz = C.c_int32(), C.c_int64()
    _check(lib.rimdp_generate_host(C.byref(cfg), C.byref(nc), C.byref(nnz), None, None, None, None, None))
    dtype = np.float64 if cfg.dtype == RIMDP_F64 else np.float32
    nst = (cfg.state_end - cfg.state_begin) if (cfg.state_begin or cfg.state_end) else cfg.num_states
    sp = np.empty(nst + 1, np.int32)
    cp = np.empty(nc.value + 1, np.int64)
    rv = np.empty(nnz.value, np.int32)
    lo = np.empty(nnz.value, dtype)
    up = np.empty(nnz.value, dtype)
    _check(lib.rimdp_generate_host(C.byref(cfg), None, None, _p(sp), _p(cp), _p(rv), _p(lo), _p(up)))
    return sp, cp, rv, lo, up


class NativeSizes(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("num_cols", C.c_int32), ("nnz", C.c_int64), ("imdp", C.c_int32),
                ("label_bytes", C.c_int64)]


def read_native_model(path, dtype=np.float64):
    """An IMDPCSC1 model container as the engine's CSC arrays (rimdp_native_read;
    the reference's io::read_native_model, io/native.hpp:457-561):
    (stateptr int32, colptr int64, rowval int32, lower, upper, labels list[str]).
    Raises EngineError with status ERR_MISSING_FILE / ERR_SCHEMA and the
    reference's message on a bad container."""
    lib = load()
    sz = NativeSizes()
    h = C.c_void_p()
    _check(lib.rimdp_native_read(os.fsencode(path), _dt(dtype), C.byref(sz), C.byref(h)))
    try:
        sp = np.empty(sz.num_states + 1, np.int32)
        cp = np.empty(sz.num_cols + 1, np.int64)
        rv = np.empty(sz.nnz, np.int32)
        lo = np.empty(sz.nnz, dtype)
        up = np.empty(sz.nnz, dtype)
        lab = C.create_string_buffer(max(int(sz.label_bytes), 1))
        _check(lib.rimdp_native_take(h, _p(sp), _p(cp), _p(rv), _p(lo), _p(up), lab))
    finally:
        lib.rimdp_native_free(h)
    labels = [x.decode() for x in lab.raw[:sz.label_bytes].split(b"\0")[:-1]]
    return sp, cp, rv, lo, up, labels


def write_native_model(path, stateptr, colptr, rowval, lower, upper, labels=None, index64=False):
    """The engine's CSC arrays as an IMDPCSC1 container (rimdp_native_write; write_native_model,
    io/native.hpp:424-455).  int64 column pointers (dtype 6) when index64 or beyond 2^31-1 transitions."""
    lower = np.asarray(lower)
    dt = lower.dtype
    sp = np.ascontiguousarray(stateptr, np.int32)
    cp = np.ascontiguousarray(colptr, np.int64)
    rv = np.ascontiguousarray(rowval, np.int32)
    lo = np.ascontiguousarray(lower, dt)
    up = np.ascontiguousarray(upper, dt)
    lab = None if labels is None else b"".join(x.encode() + b"\0" for x in labels)
    _check(load().rimdp_native_write(os.fsencode(path), _dt(dt), len(sp) - 1, len(cp) - 1, _p(sp), _p(cp), _p(rv),
                                     _p(lo), _p(up), lab, int(bool(index64))))


def _dt(dtype) -> int:
    return RIMDP_F64 if np.dtype(dtype) == np.float64 else RIMDP_F32


def _p(a):
    return None if a is None else a.ctypes.data


class DeviceModel:
    """A transition store resident in HBM (rimdp_model)."""

    def __init__(self, handle, dtype):
        self._h = handle
        self.dtype = np.dtype(dtype)
        self._keep = []
        inf = self.info()
        self.num_states = inf.num_states
        self.num_cols = inf.num_cols
        self.nnz = inf.nnz
        self.state_begin = inf.state_begin
        self.state_end = inf.state_end

    @classmethod
    def from_csc(cls, stateptr, colptr, rowval, lower, upper, device: int = 0) -> "DeviceModel":
        lower = np.asarray(lower)
        dtype = lower.dtype
        if dtype not in (np.float64, np.float32):
            raise TypeError("lower/upper must be float64 or float32")
        sp = np.ascontiguousarray(stateptr, np.int32)
        cp = np.ascontiguousarray(colptr, np.int64)
        rv = np.ascontiguousarray(rowval, np.int32)
        lo = np.ascontiguousarray(lower, dtype)
        up = np.ascontiguousarray(upper, dtype)
        d = ModelDesc(_dt(dtype), device, len(sp) - 1, len(cp) - 1, int(cp[-1]), _p(sp), _p(cp), _p(rv), _p(lo), _p(up))
        h = C.c_void_p()
        _check(load().rimdp_model_create(C.byref(d), C.byref(h)))
        return cls(h, dtype)

    @classmethod
    def from_csc_shard(cls, stateptr, colptr, rowval, lower, upper, state_begin: int, num_global_states: int,
                       device: int = 0) -> "DeviceModel":
        """One shard: local stateptr/colptr (rebased to 0), global destination rows."""
        lower = np.asarray(lower)
        dtype = lower.dtype
        sp = np.ascontiguousarray(stateptr, np.int32)
        cp = np.ascontiguousarray(colptr, np.int64)
        rv = np.ascontiguousarray(rowval, np.int32)
        lo = np.ascontiguousarray(lower, dtype)
        up = np.ascontiguousarray(upper, dtype)
        d = ModelDesc(_dt(dtype), device, len(sp) - 1, len(cp) - 1, int(cp[-1]), _p(sp), _p(cp), _p(rv), _p(lo), _p(up))
        h = C.c_void_p()
        _check(load().rimdp_model_create_shard(C.byref(d), int(state_begin), int(num_global_states), C.byref(h)))
        return cls(h, dtype)

    @classmethod
    def from_native(cls, path, dtype=np.float64, device: int = 0) -> "DeviceModel":
        """Upload an IMDPCSC1 container's CSC arrays directly."""
        sp, cp, rv, lo, up, _ = read_native_model(path, dtype)
        return cls.from_csc(sp, cp, rv, lo, up, device=device)

    @classmethod
    def generate(cls, cfg: GenConfig) -> "DeviceModel":
        h = C.c_void_p()
        _check(load().rimdp_model_generate(C.byref(cfg), C.byref(h)))
        return cls(h, np.float64 if cfg.dtype == RIMDP_F64 else np.float32)

    def read_columns(self, col_begin: int, col_end: int):
        """(colptr int64 relative, rows int32, lower, gap) of columns [col_begin, col_end) as stored."""
        cp = np.empty(col_end - col_begin + 1, np.int64)
        _check(load().rimdp_model_read_columns(self._h, col_begin, col_end, _p(cp), None, None, None))
        cnt = int(cp[-1])
        rv = np.empty(cnt, np.int32)
        lo = np.empty(cnt, self.dtype)
        gp = np.empty(cnt, self.dtype)
        _check(load().rimdp_model_read_columns(self._h, col_begin, col_end, _p(cp), _p(rv), _p(lo), _p(gp)))
        return cp, rv, lo, gp

    def close(self):
        if getattr(self, "_h", None):
            load().rimdp_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> ModelInfo:
        i = ModelInfo()
        _check(load().rimdp_model_info_get(self._h, C.byref(i)))
        return i

    def stream(self) -> int:
        s = C.c_void_p()
        _check(load().rimdp_model_stream(self._h, C.byref(s)))
        return s.value or 0

    # -- plans ---------------------------------------------------------------
    def _plan(self, *, initial, pessimistic=True, maximize=True, finite=True, horizon=0, eps=0.0,
              max_iterations=1_000_000, frozen=None, rewards=None, discount=0.0, forced=None, external_stop=False):
        keep = []
        n = self.num_states if self.state_end - self.state_begin == self.num_states else None
        v0 = np.ascontiguousarray(initial, self.dtype)
        keep.append(v0)
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.uint8)
        rw = None if rewards is None else np.ascontiguousarray(rewards, self.dtype)
        fc = None if forced is None else np.ascontiguousarray(forced, np.int32)
        keep += [fz, rw, fc]
        del n
        plan = Plan(int(bool(pessimistic)), int(bool(maximize)), int(bool(finite)), int(horizon), float(eps),
                    int(max_iterations), _p(v0), _p(fz), _p(rw), float(discount), _p(fc),
                    int(fc is not None and fc.ndim == 2), int(bool(external_stop)))
        return plan, keep

    def solve(self, *, record="none", on_iteration=None, **kw):
        """Full solve.  record: "none" | "last" | "all" (per-step chosen columns)."""
        plan, keep = self._plan(**kw)
        nv = len(keep[0])
        values = np.empty(nv, self.dtype)
        residual = np.empty(nv, self.dtype)
        it = C.c_int64()
        chosen = None
        if record == "last":
            chosen = np.empty(self.state_end - self.state_begin, np.int32)
        elif record == "all":
            chosen = np.empty((max(int(kw.get("horizon", 0)), 0), self.state_end - self.state_begin), np.int32)
        cb = ITER_CB()
        if on_iteration is not None:
            dt, n = self.dtype, nv

            def _cb(k, vals, user):
                arr = np.ctypeslib.as_array(C.cast(vals, C.POINTER(C.c_double if dt == np.float64 else C.c_float)),
                                            shape=(n,)).copy()
                on_iteration(int(k), arr)

            cb = ITER_CB(_cb)
        out = Outputs(values.ctypes.data, residual.ctypes.data, C.pointer(it), _p(chosen),
                      int(record == "all"), cb, None)
        _check(load().rimdp_solve(self._h, C.byref(plan), C.byref(out)))
        res = {"values": values, "residual": residual, "iterations": it.value}
        if chosen is not None:
            res["chosen"] = chosen
        return res

    def bellman_step(self, values, pessimistic=True, maximize=True, frozen=None, forced=None):
        v = np.ascontiguousarray(values, self.dtype)
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.uint8)
        fc = None if forced is None else np.ascontiguousarray(forced, np.int32)
        out = np.empty(len(v), self.dtype)
        ch = np.empty(self.state_end - self.state_begin, np.int32)
        _check(load().rimdp_bellman_step(self._h, _p(v), int(bool(pessimistic)), int(bool(maximize)), _p(fz), _p(fc),
                                         _p(out), _p(ch)))
        return out, ch

    def column_values(self, values, pessimistic=True):
        v = np.ascontiguousarray(values, self.dtype)
        q = np.empty(self.num_cols, self.dtype)
        _check(load().rimdp_column_values(self._h, _p(v), int(bool(pessimistic)), _p(q)))
        return q

    # -- split solve (resident benchmarking / sharded driver) ---------------
    def begin(self, **kw):
        plan, keep = self._plan(**kw)
        self._keep = keep
        _check(load().rimdp_solve_begin(self._h, C.byref(plan)))

    def advance(self, iterations: int):
        _check(load().rimdp_solve_advance(self._h, C.c_int64(iterations)))

    def poll(self):
        k, fin, res = C.c_int64(), C.c_int32(), C.c_double()
        _check(load().rimdp_solve_poll(self._h, C.byref(k), C.byref(fin), C.byref(res)))
        return k.value, bool(fin.value), res.value

    def finish(self, record=False):
        nv = len(self._keep[0])
        values = np.empty(nv, self.dtype)
        residual = np.empty(nv, self.dtype)
        it = C.c_int64()
        out = Outputs(values.ctypes.data, residual.ctypes.data, C.pointer(it), None, 0, ITER_CB(), None)
        _check(load().rimdp_solve_finish(self._h, C.byref(out)))
        return {"values": values, "residual": residual, "iterations": it.value}

    def profile(self, on: bool = True):
        _check(load().rimdp_profile_enable(self._h, int(on)))

    def profile_read(self):
        """Summed ms of (fused short-state kernel, per-column kernels, action kernel), iterations,
        kernels per iteration — since the last read."""
        f, c, a, it, kp = C.c_double(), C.c_double(), C.c_double(), C.c_int64(), C.c_int32()
        _check(load().rimdp_profile_read(self._h, C.byref(f), C.byref(c), C.byref(a), C.byref(it), C.byref(kp)))
        return f.value, c.value, a.value, it.value, kp.value

    def set_value_capacity(self, entries: int):
        _check(load().rimdp_model_set_value_capacity(self._h, int(entries)))

    def residual_slots(self) -> int:
        p = C.c_void_p()
        _check(load().rimdp_solve_residual_slots(self._h, C.byref(p)))
        return p.value

    def stop_test(self):
        _check(load().rimdp_solve_stop_test(self._h))

    # -- peer exchange (state-sharded solves across processes) ---------------
    def exchange_export(self) -> bytes:
        """This shard's exchange window as a 64-byte CUDA IPC handle (rimdp_exchange_export)."""
        h = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(load().rimdp_exchange_export(self._h, h))
        return h.raw

    def exchange_connect(self, rank: int, world: int, handles: list) -> None:
        """Map every rank's window (rank order, as exported) into this shard's peer table."""
        blob = b"".join(handles)
        if len(blob) != IPC_HANDLE_BYTES * world:
            raise ValueError("one 64-byte handle per rank is required")
        _check(load().rimdp_exchange_connect(self._h, int(rank), int(world), blob))

    def value_buffers(self):
        b0, b1 = C.c_void_p(), C.c_void_p()
        _check(load().rimdp_solve_value_buffers(self._h, C.byref(b0), C.byref(b1)))
        return b0.value, b1.value


IPC_HANDLE_BYTES = 64


def connect_local(shards) -> None:
    """Shards of one model in this process (devices may repeat): rimdp_exchange_connect_local."""
    arr = (C.c_void_p * len(shards))(*[m._h.value if isinstance(m._h, C.c_void_p) else m._h for m in shards])
    _check(load().rimdp_exchange_connect_local(arr, len(shards)))


class MultiModel:
    """A model cut into state shards on several devices of this process, exchanging V over peer
    memory (rimdp_multi_*).  Same solve surface as DeviceModel (global columns, whole vectors)."""

    def __init__(self, stateptr, colptr, rowval, lower, upper, world: int, devices=None):
        lower = np.asarray(lower)
        self.dtype = np.dtype(lower.dtype)
        sp = np.ascontiguousarray(stateptr, np.int32)
        cp = np.ascontiguousarray(colptr, np.int64)
        rv = np.ascontiguousarray(rowval, np.int32)
        lo = np.ascontiguousarray(lower, self.dtype)
        up = np.ascontiguousarray(upper, self.dtype)
        d = ModelDesc(_dt(self.dtype), 0, len(sp) - 1, len(cp) - 1, int(cp[-1]), _p(sp), _p(cp), _p(rv), _p(lo), _p(up))
        dev = None if devices is None else np.ascontiguousarray(devices, np.int32)
        self._h = C.c_void_p()
        _check(load().rimdp_multi_create(C.byref(d), int(world), _p(dev), C.byref(self._h)))
        self.num_states = len(sp) - 1
        self.num_cols = len(cp) - 1
        self.nnz = int(cp[-1])
        self.state_begin, self.state_end = 0, self.num_states
        self.world = int(world)

    def info(self):
        w = C.c_int32()
        sb = np.empty(self.world + 1, np.int32)
        dv = np.empty(self.world, np.int32)
        _check(load().rimdp_multi_info(self._h, C.byref(w), _p(sb), _p(dv)))
        return {"world": w.value, "state_begin": sb, "devices": dv}

    def close(self):
        if getattr(self, "_h", None):
            load().rimdp_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    _plan = DeviceModel._plan

    def solve(self, *, record="none", on_iteration=None, **kw):
        plan, keep = self._plan(**kw)
        n = self.num_states
        values = np.empty(n, self.dtype)
        residual = np.empty(n, self.dtype)
        it = C.c_int64()
        chosen = None
        if record == "last":
            chosen = np.empty(n, np.int32)
        elif record == "all":
            chosen = np.empty((max(int(kw.get("horizon", 0)), 0), n), np.int32)
        cb = ITER_CB()
        if on_iteration is not None:
            dt = self.dtype

            def _cb(k, vals, user):
                arr = np.ctypeslib.as_array(C.cast(vals, C.POINTER(C.c_double if dt == np.float64 else C.c_float)),
                                            shape=(n,)).copy()
                on_iteration(int(k), arr)

            cb = ITER_CB(_cb)
        out = Outputs(values.ctypes.data, residual.ctypes.data, C.pointer(it), _p(chosen), int(record == "all"), cb,
                      None)
        _check(load().rimdp_multi_solve(self._h, C.byref(plan), C.byref(out)))
        res = {"values": values, "residual": residual, "iterations": it.value}
        if chosen is not None:
            res["chosen"] = chosen
        return res
