"""Device-side model validation at upload: broken CSC
arrays given to the raw C ABI (rimdp_model_create) are rejected with the
reference's first violation — the same ViolationKind, column, row and
ModelError text that the reference's checked constructor
(IntervalProbabilities::from_aligned -> validate, interval.hpp:67-77,
132-179; CscMatrix::structural_violation, csc.hpp:75-107) raises on the same
arrays (oracle/_ref)."""
import numpy as np
import pytest

import oracle
from paper_2401_04068_b200 import engine

pytestmark = pytest.mark.gpu


def base(dtype=np.float64):
    return [a.copy() for a in engine.random_imdp(40, 3, 0.25, 0.2, 11, dtype=dtype)]


def entry(cp, col, k):
    return int(cp[col]) + k


def mutate(kind, arrays):
    sp, cp, rv, lo, up = arrays
    if kind == "rows_unsorted":
        i = entry(cp, 7, 1)
        rv[i - 1], rv[i] = rv[i], rv[i - 1]
    elif kind == "row_out_of_range":
        rv[entry(cp, 30, 2)] = 40
    elif kind == "row_negative":
        rv[entry(cp, 5, 0)] = -1
    elif kind == "lower_nan":
        lo[entry(cp, 12, 1)] = np.nan
    elif kind == "upper_above_one":
        up[entry(cp, 3, 2)] = 1.5
    elif kind == "lower_negative":
        lo[entry(cp, 9, 0)] = -0.25
    elif kind == "upper_inf":
        up[entry(cp, 2, 1)] = np.inf
    elif kind == "lower_exceeds_upper":
        i = entry(cp, 20, 1)
        lo[i], up[i] = 0.3, 0.2
    elif kind == "lower_positive_upper_zero":
        i = entry(cp, 21, 0)
        lo[i], up[i] = 0.1, 0.0
    elif kind == "first_of_several":
        # column 3: upper > 1 at its third entry; column 1: lower and upper out of range at one entry
        # (the lower bound is reported); column 25: unsorted rows — structure is checked first
        up[entry(cp, 3, 2)] = 2.0
        i = entry(cp, 1, 1)
        lo[i], up[i] = 1.5, 3.0
        j = entry(cp, 25, 1)
        rv[j - 1], rv[j] = rv[j], rv[j - 1]
    elif kind == "entries_before_sums":
        # column 4 only infeasible (sums), column 6 an entry violation: the entry one is what upload rejects
        up[cp[4]:cp[5]] = lo[cp[4]:cp[5]]
        lo[entry(cp, 6, 0)] = 2.0
    return sp, cp, rv, lo, up


KINDS = ["rows_unsorted", "row_out_of_range", "row_negative", "lower_nan", "upper_above_one", "lower_negative",
         "upper_inf", "lower_exceeds_upper", "lower_positive_upper_zero", "first_of_several",
         "entries_before_sums"]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("kind", KINDS)
def test_upload_rejects_broken_arrays_like_the_reference(kind, dtype):
    arrays = mutate(kind, base(dtype))
    with pytest.raises(oracle.OracleError) as ref:
        oracle.Model.from_arrays("ref", *arrays, checked=True)
    with pytest.raises(engine.EngineError) as dev:
        engine.DeviceModel.from_csc(*arrays)
    e, r = dev.value, ref.value
    assert e.status == engine.ERR_INVALID_MODEL, e.message
    if kind == "entries_before_sums":
        # the reference reports column 4's InfeasibleColumn first; upload leaves sums to the step
        assert r.violation_kind == 3 and e.violation_kind == 1 and e.column == 6
        return
    assert e.message == r.message
    assert e.violation_kind == r.violation_kind
    assert engine.VIOLATION_KINDS[e.violation_kind] == e.message.split(" ")[0]


def test_valid_and_infeasible_models_still_upload():
    sp, cp, rv, lo, up = base()
    engine.DeviceModel.from_csc(sp, cp, rv, lo, up).close()
    up = up.copy()
    up[cp[4]:cp[5]] = lo[cp[4]:cp[5]]   # infeasible column: reported when a step evaluates it
    m = engine.DeviceModel.from_csc(sp, cp, rv, lo, up)
    assert m.info().num_infeasible_columns == 1
    m.close()


def test_multi_model_reports_global_columns():
    arrays = mutate("upper_above_one", base())
    arrays[3][engine.random_imdp(40, 3, 0.25, 0.2, 11)[1][35]] = -1.0  # column 35 too (a later shard)
    with pytest.raises(engine.EngineError) as single:
        engine.DeviceModel.from_csc(*arrays)
    arrays2 = list(base())
    cp = arrays2[1]
    arrays2[3][cp[35]] = -1.0
    with pytest.raises(engine.EngineError) as multi:
        engine.MultiModel(*arrays2, world=2, devices=[0, 0])
    assert single.value.column == 3
    assert multi.value.column == 35 and "column=35" in multi.value.message
