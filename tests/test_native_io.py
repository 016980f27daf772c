"""Native IMDPCSC1 containers -> the engine's CSC arrays.

rimdp_native_read is host code in the engine library (csrc/native_io.cpp), so
these run on CPU.  Every case is checked against the reference's own
io::read_native_model (io/native.hpp:457-561) compiled in oracle/_ref:
identical arrays and labels for valid containers, and the identical
exception text for broken ones (SchemaViolation / MissingFile, errors.hpp).
"""
from __future__ import annotations

import os
import struct

import numpy as np
import pytest

import oracle
from paper_2401_04068_b200 import engine

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")


def _str(s: str) -> bytes:
    b = s.encode()
    return struct.pack("<I", len(b)) + b


def write_container(path, attrs: dict, variables: dict):
    """The binary container layout of io/native.hpp:252-293 (test-side writer).
    variables: name -> (dtype code, payload) with 1 int32, 2 f64, 3 f32, 4 strings."""
    out = bytearray(b"IMDPCSC1")
    out += struct.pack("<I", len(attrs))
    for k, v in attrs.items():
        out += _str(k) + _str(v)
    out += struct.pack("<I", len(variables))
    for k, (code, data) in variables.items():
        out += _str(k) + struct.pack("<B", code) + struct.pack("<Q", len(data))
        if code == 1:
            out += np.asarray(data, "<i4").tobytes()
        elif code == 2:
            out += np.asarray(data, "<f8").tobytes()
        elif code == 3:
            out += np.asarray(data, "<f4").tobytes()
        else:
            for s in data:
                out += _str(s)
    with open(path, "wb") as f:
        f.write(bytes(out))


def paper_container(**over):
    """The paper's 3-state IMDP (test_solver.cpp:13-25) as separate lower/upper CSC matrices."""
    lower = [[0.0, 0.1, 0.2], [0.5, 0.3, 0.1], [0.1, 0.2, 0.3], [0.2, 0.3, 0.4], [0.0, 0.0, 1.0]]
    upper = [[0.5, 0.6, 0.7], [0.7, 0.5, 0.3], [0.6, 0.5, 0.4], [0.6, 0.5, 0.4], [0.0, 0.0, 1.0]]

    def csc(m):
        cp, rv, nz = [0], [], []
        for col in m:
            for r, x in enumerate(col):
                if x != 0.0:
                    rv.append(r)
                    nz.append(x)
            cp.append(len(rv))
        return cp, rv, nz

    lcp, lrv, lnz = csc(lower)
    ucp, urv, unz = csc(upper)
    attrs = {"model": "imdp", "format": "sparse_csc", "rows": "to", "cols": "from/action", "num_states": "3"}
    var = {"lower_colptr": (1, lcp), "lower_rowval": (1, lrv), "lower_nzval": (2, lnz),
           "upper_colptr": (1, ucp), "upper_rowval": (1, urv), "upper_nzval": (2, unz),
           "stateptr": (1, [0, 2, 4, 5]), "action_vals": (4, ["a1", "a2", "a1", "a2", "sink"])}
    for k, v in over.items():
        if k.startswith("attr_"):
            if v is None:
                attrs.pop(k[5:])
            else:
                attrs[k[5:]] = v
        elif v is None:
            var.pop(k)
        else:
            var[k] = v
    return attrs, var


def both(path, dtype=np.float64):
    """(ours, reference): arrays or the error text."""
    try:
        mine = engine.read_native_model(path, dtype)
    except engine.EngineError as e:
        mine = ("error", e.status, e.message)
    try:
        m = oracle.Model.read_native(path, dtype)
        sp, cp, rv, lo, up = m.export()
        ref = (sp, cp, rv, lo, up, m.labels())
    except oracle.OracleError as e:
        ref = ("error", str(e))
    return mine, ref


def assert_same_model(mine, ref):
    assert not isinstance(mine[0], str) and not isinstance(ref[0], str), (mine, ref)
    for a, b in zip(mine[:5], ref[:5]):
        assert a.dtype.kind == b.dtype.kind
        assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b, a.dtype).view(np.uint8))
    assert mine[5] == ref[5]


def assert_same_error(mine, ref):
    assert mine[0] == "error" and ref[0] == "error", (mine, ref)
    assert mine[1] in (engine.ERR_SCHEMA, engine.ERR_MISSING_FILE)
    assert mine[2] in ref[1], (mine[2], ref[1])


@needs_ref
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("seed", [1, 7])
def test_reference_written_random_models_read_identically(tmp_path, dtype, seed):
    m = oracle.Model.random(300, 3, 0.05, 0.04, seed, dtype=dtype)
    path = str(tmp_path / "m.imdpcsc")
    m.write_native(path)
    mine, ref = both(path, dtype)
    assert_same_model(mine, ref)
    sp, cp, rv, lo, up = m.export()
    assert np.array_equal(mine[1], cp) and np.array_equal(mine[3], lo)


@needs_ref
def test_paper_container_aligns_and_drops_empty_intervals(tmp_path):
    path = str(tmp_path / "p.imdpcsc")
    write_container(path, *paper_container())
    mine, ref = both(path)
    assert_same_model(mine, ref)
    # the [0,0] entries of the sink column and of column 0's row 0 lower bound
    assert list(mine[1]) == [0, 3, 6, 9, 12, 13]
    assert mine[5] == ["a1", "a2", "a1", "a2", "sink"]


@needs_ref
def test_f32_container_promotes_into_f64_store(tmp_path):
    attrs, var = paper_container()
    var["lower_nzval"] = (3, var["lower_nzval"][1])
    var["upper_nzval"] = (3, var["upper_nzval"][1])
    path = str(tmp_path / "p.imdpcsc")
    write_container(path, attrs, var)
    for dtype in (np.float64, np.float32):
        mine, ref = both(path, dtype)
        assert_same_model(mine, ref)
    # mixed: the f32-rounded lower bound 0.4 exceeds the f64 upper bound 0.4 (a BoundOrderViolation)
    var["upper_nzval"] = (2, var["upper_nzval"][1])
    write_container(path, attrs, var)
    assert_same_error(*both(path, np.float64))
    # an f32 store refuses f64 data (NativeValueCodec<float>::unpack, native.hpp:219-225)
    assert_same_error(*both(path, np.float32))


@needs_ref
def test_imc_container_promotes_to_one_action_per_state(tmp_path):
    attrs = {"model": "imc", "format": "sparse_csc", "rows": "to", "cols": "from", "num_states": "2"}
    var = {"lower_colptr": (1, [0, 1, 2]), "lower_rowval": (1, [0, 1]), "lower_nzval": (2, [0.2, 1.0]),
           "upper_colptr": (1, [0, 2, 3]), "upper_rowval": (1, [0, 1, 1]), "upper_nzval": (2, [0.5, 0.8, 1.0])}
    path = str(tmp_path / "c.imdpcsc")
    write_container(path, attrs, var)
    mine, ref = both(path)
    assert_same_model(mine, ref)
    assert mine[5] == ["0", "0"]


BROKEN = {
    "model": dict(attr_model="mdp"),
    "format": dict(attr_format="dense"),
    "rows": dict(attr_rows="from"),
    "cols": dict(attr_cols="from"),
    "num_states": dict(attr_num_states="x3"),
    "num_states_missing": dict(attr_num_states=None),
    "missing_var": dict(upper_rowval=None),
    "int_type": dict(stateptr=(2, [0.0, 2.0, 4.0, 5.0])),
    "labels_type": dict(action_vals=(1, [0, 1, 0, 1, 0])),
    "nz_type": dict(lower_nzval=(1, [1] * 11)),
    "col_count": dict(lower_colptr=(1, [0, 2, 5, 8, 11])),
    "row_oob": dict(upper_rowval=(1, [0, 1, 2, 0, 1, 2, 0, 1, 2, 0, 1, 3, 2])),
    "colptr_start": dict(upper_colptr=(1, [1, 3, 6, 9, 12, 13])),
    "colptr_end": dict(upper_colptr=(1, [0, 3, 6, 9, 12, 12])),
    "colptr_monotone": dict(upper_colptr=(1, [0, 3, 2, 9, 12, 13])),
    "rows_order": dict(upper_rowval=(1, [0, 2, 1, 0, 1, 2, 0, 1, 2, 0, 1, 2, 2])),
    "entry_range": dict(upper_nzval=(2, [0.5, 0.6, 1.7, 0.7, 0.5, 0.3, 0.6, 0.5, 0.4, 0.6, 0.5, 0.4, 1.0])),
    "entry_nan": dict(upper_nzval=(2, [0.5, 0.6, float("nan"), 0.7, 0.5, 0.3, 0.6, 0.5, 0.4, 0.6, 0.5, 0.4, 1.0])),
    "order": dict(upper_nzval=(2, [0.5, 0.6, 0.7, 0.7, 0.2, 0.3, 0.6, 0.5, 0.4, 0.6, 0.5, 0.4, 1.0])),
    "lower_sum": dict(lower_nzval=(2, [0.1, 0.2, 0.5, 0.3, 0.1, 0.1, 0.2, 0.3, 0.5, 0.3, 0.4])),
    "upper_sum": dict(upper_nzval=(2, [0.5, 0.6, 0.7, 0.7, 0.5, 0.3, 0.3, 0.3, 0.3, 0.6, 0.5, 0.4, 1.0])),
    "stateptr_start": dict(stateptr=(1, [1, 2, 4, 5])),
    "stateptr_states": dict(stateptr=(1, [0, 2, 5])),
    "stateptr_end": dict(stateptr=(1, [0, 2, 3, 4])),
    "label_count": dict(action_vals=(4, ["a1", "a2", "a1", "a2"])),
    "empty_action_set": dict(stateptr=(1, [0, 2, 2, 5]), action_vals=(4, ["a", "b", "c", "d", "e"])),
    "duplicate_label": dict(action_vals=(4, ["a1", "a1", "a1", "a2", "sink"])),
}


@pytest.mark.parametrize("case", sorted(BROKEN))
@needs_ref
def test_broken_containers_fail_like_the_reference(tmp_path, case):
    path = str(tmp_path / f"{case}.imdpcsc")
    write_container(path, *paper_container(**BROKEN[case]))
    mine, ref = both(path)
    assert_same_error(mine, ref)


@needs_ref
def test_truncated_and_missing_files(tmp_path):
    path = str(tmp_path / "p.imdpcsc")
    write_container(path, *paper_container())
    data = open(path, "rb").read()
    for cut in (12, 40, len(data) - 3):
        with open(path, "wb") as f:
            f.write(data[:cut])
        assert_same_error(*both(path))
    missing = str(tmp_path / "nope.imdpcsc")
    mine, ref = both(missing)
    assert_same_error(mine, ref)
    assert mine[1] == engine.ERR_MISSING_FILE


@needs_ref
def test_json_debug_variant_is_refused_with_a_schema_violation(tmp_path):
    """The JSON debug container (native.hpp:349-421) is text parsing, out of
    scope for the engine's reader: it is refused loudly, never misread."""
    m = oracle.Model.random(20, 2, 0.3, 0.2, 3)
    path = str(tmp_path / "m.json")
    m.write_native(path, json_debug=True)
    with pytest.raises(engine.EngineError) as e:
        engine.read_native_model(path)
    assert e.value.status == engine.ERR_SCHEMA
    assert os.path.exists(path)


@pytest.mark.gpu
def test_native_container_uploads_and_solves_like_the_golden_arrays(tmp_path, golden):
    """Container -> rimdp_native_read -> rimdp_model_create -> solve: bit-exact
    against the reference's golden solves of the same models (no reference
    needed on the box: the container is written by the test-side writer)."""
    from paper_2401_04068_b200 import problems as P
    from test_engine_gpu import bits, spec_from

    for name in golden.models():
        sp, cp, rv, lo, up = golden.model(name)
        n = len(sp) - 1
        cp32 = [int(x) for x in cp]
        attrs = {"model": "imdp", "format": "sparse_csc", "rows": "to", "cols": "from/action", "num_states": str(n)}
        code = 2 if lo.dtype == np.float64 else 3
        var = {"lower_colptr": (1, cp32), "lower_rowval": (1, rv), "lower_nzval": (code, lo),
               "upper_colptr": (1, cp32), "upper_rowval": (1, rv), "upper_nzval": (code, up),
               "stateptr": (1, sp), "action_vals": (4, [str(i) for i in range(len(cp) - 1)])}
        path = str(tmp_path / f"{name}.imdpcsc")
        write_container(path, attrs, var)
        m = engine.DeviceModel.from_native(path, dtype=lo.dtype)
        assert (m.num_states, m.num_cols, m.nnz) == (n, len(cp) - 1, int(cp[-1]))
        for key in golden.solves(name):
            meta = golden.meta[key]
            if not meta["ok"]:
                continue
            policy, vf = P.control_synthesis(m, spec_from(meta, golden, key), sp,
                                             max_iterations=meta["max_iterations"])
            assert vf.iterations == meta["iterations"], key
            assert np.array_equal(bits(vf.values), bits(golden.get(f"{key}/values"))), key
            assert np.array_equal(policy.columns, golden.get(f"{key}/policy")), key
        m.close()


# ---- the writer and the 64-bit column pointers (dtype 6) ----------------------------------------

@needs_ref
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_writer_is_byte_identical_to_the_reference_writer(tmp_path, dtype):
    """rimdp_native_write with int32 pointers == write_native_model (native.hpp:424-455), byte for byte."""
    m = oracle.Model.random(300, 3, 0.05, 0.04, 5, dtype=dtype)
    a, b = str(tmp_path / "ref.imdpcsc"), str(tmp_path / "mine.imdpcsc")
    m.write_native(a)
    engine.write_native_model(b, *m.export(), labels=m.labels())
    assert open(a, "rb").read() == open(b, "rb").read()


@needs_ref
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_int64_column_pointers_round_trip(tmp_path, dtype):
    m = oracle.Model.random(250, 4, 0.06, 0.05, 9, dtype=dtype)
    arrays = m.export()
    path = str(tmp_path / "wide.imdpcsc")
    engine.write_native_model(path, *arrays, labels=m.labels(), index64=True)
    raw = open(path, "rb").read()
    assert raw.count(b"lower_colptr\x06") == 1 and raw.count(b"upper_colptr\x06") == 1  # dtype 6 = int64
    sp, cp, rv, lo, up, labels = engine.read_native_model(path, dtype)
    for x, y in zip((sp, cp, rv, lo, up), arrays):
        assert np.array_equal(np.asarray(x), np.asarray(y)) and np.asarray(x).dtype.kind == np.asarray(y).dtype.kind
    assert labels == m.labels()
    # the reference's reader does not know the extension (native.hpp:340-341: unknown dtype)
    with pytest.raises(oracle.OracleError) as e:
        oracle.Model.read_native(path, dtype)
    assert "unknown dtype 6" in e.value.message


def test_int64_container_structure_is_checked(tmp_path):
    attrs = {"model": "imdp", "format": "sparse_csc", "rows": "to", "cols": "from/action", "num_states": "2"}

    def wide(path, cp):
        out = bytearray(b"IMDPCSC1") + struct.pack("<I", len(attrs))
        for k, v in attrs.items():
            out += _str(k) + _str(v)
        variables = [("lower_colptr", cp), ("upper_colptr", cp)]
        out += struct.pack("<I", 8)
        for k, p in variables:
            out += _str(k) + struct.pack("<BQ", 6, len(p)) + np.asarray(p, "<i8").tobytes()
        for k, code, data in (("lower_rowval", 1, [0, 1, 1]), ("upper_rowval", 1, [0, 1, 1]),
                              ("lower_nzval", 2, [0.2, 0.3, 0.5]), ("upper_nzval", 2, [0.6, 0.8, 1.0]),
                              ("stateptr", 1, [0, 1, 2])):
            out += _str(k) + struct.pack("<BQ", code, len(data))
            out += np.asarray(data, "<i4" if code == 1 else "<f8").tobytes()
        out += _str("action_vals") + struct.pack("<BQ", 4, 2) + _str("a") + _str("b")
        with open(path, "wb") as f:
            f.write(bytes(out))

    good = str(tmp_path / "good.imdpcsc")
    wide(good, [0, 2, 3])
    sp, cp, rv, lo, up, labels = engine.read_native_model(good)
    assert list(cp) == [0, 2, 3] and labels == ["a", "b"]
    bad = str(tmp_path / "bad.imdpcsc")
    wide(bad, [0, 2 ** 40, 3])  # a middle pointer far past the row array
    with pytest.raises(engine.EngineError) as e:
        engine.read_native_model(bad)
    assert e.value.status == engine.ERR_SCHEMA and "colptr not monotone" in e.value.message


@pytest.mark.gpu
@needs_ref
def test_int64_container_uploads_and_solves_bit_exact(tmp_path):
    from paper_2401_04068_b200 import problems as P
    m = oracle.Model.random(400, 3, 24.0 / 400, 1.0 / 24, 3)
    arrays = m.export()
    path = str(tmp_path / "wide.imdpcsc")
    engine.write_native_model(path, *arrays, index64=True)
    dev = engine.DeviceModel.from_native(path)
    spec = P.Specification(P.InfiniteTimeReachability(list(range(390, 400)), 1e-6))
    pol, vf = P.control_synthesis(dev, spec, arrays[0])
    ref = m.solve(oracle.Problem(oracle.INFINITE_REACH, reach=list(range(390, 400)), eps=1e-6), synthesize=True)
    assert vf.iterations == ref["iterations"]
    assert np.array_equal(vf.values.view(np.uint64), ref["values"].view(np.uint64))
    assert np.array_equal(pol.columns, ref["policy"])
