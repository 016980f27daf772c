"""Pin the CPU checkers: the plain-C restatement (oracle/port) and, when the
reference is present, the reference library (oracle/_ref) must reproduce the
golden fixtures bit for bit, and the SURVEY Appendix A known answers."""
import numpy as np
import pytest

import oracle
from oracle import Model, Problem

APPENDIX_A = {  # (V0 bits, V1 bits, policy s0, policy s1) at K=10
    (1, 1): (0x3feeb672f1a3c19a, 0x3fef12791ba33345),
    (1, 0): (0x3fefff5b12c0e4f1, 0x3feffeb62581c9e3),
    (0, 1): (0x3fea4777fdc61c8b, 0x3feb807087791bf8),
    (0, 0): (0x3feeea50d1a63bc3, 0x3fef46e07970e7f1),
}


@pytest.fixture(scope="module", autouse=True)
def _build():
    oracle.build()


def problem_from(meta, g, key):
    m = meta
    return Problem(m["kind"], reach=m["reach"], avoid=m["avoid"], rewards=g.get(f"{key}/rewards"),
                   discount=m["discount"], horizon=m["horizon"], eps=m["eps"], pessimistic=bool(m["pessimistic"]),
                   maximize=bool(m["maximize"]), max_iterations=m["max_iterations"])


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def check_solve(which, g, key):
    meta = g.meta[key]
    name = key.split("/")[0]
    m = Model.from_arrays(which, *g.model(name))
    pr = problem_from(meta, g, key)
    if not meta["ok"]:
        with pytest.raises(oracle.OracleError) as ei:
            m.solve(pr, synthesize=True)
        assert ei.value.kind == meta["error"]
        assert ei.value.iterations == meta["iterations"]
        return
    out = m.solve(pr, synthesize=True)
    assert out["iterations"] == meta["iterations"], key
    assert np.array_equal(bits(out["values"]), bits(g.get(f"{key}/values"))), key
    assert np.array_equal(bits(out["residual"]), bits(g.get(f"{key}/residual"))), key
    assert np.array_equal(np.asarray(out["policy"]), g.get(f"{key}/policy")), key


def test_port_reproduces_every_golden_solve(golden):
    for key in golden.solves():
        check_solve("port", golden, key)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built here")
def test_reference_reproduces_every_golden_solve(golden):
    for key in golden.solves():
        if key.split("/")[0] in ("paper", "r15s1", "r200l", "f32r60"):
            check_solve("ref", golden, key)


def test_appendix_a_known_answers(golden):
    m = Model.from_arrays("port", *golden.model("paper"))
    for (mx, pe), (b0, b1) in APPENDIX_A.items():
        out = m.solve(Problem(oracle.FINITE_REACH, reach=[2], horizon=10, pessimistic=pe, maximize=mx),
                      synthesize=True)
        assert bits(out["values"])[0] == b0 and bits(out["values"])[1] == b1
        assert out["values"][2] == 1.0
        assert (out["policy"][2] == 4).all()  # the sink's only column
    # min/opt: state 1 switches to a1 (column 2) at t = 9 only
    out = m.solve(Problem(oracle.FINITE_REACH, reach=[2], horizon=10, pessimistic=False, maximize=False),
                  synthesize=True)
    assert list(out["policy"][1]) == [3] * 9 + [2]


def test_appendix_a_one_step(golden):
    m = Model.from_arrays("port", *golden.model("paper"))
    expect = {(1, 1): ([0.2, 0.4, 1], [0, 3, -1]), (1, 0): ([0.7, 0.4, 1], [0, 2, -1]),
              (0, 1): ([0.1, 0.3, 1], [1, 2, -1]), (0, 0): ([0.19999999999999998, 0.4, 1], [1, 2, -1])}
    for (mx, pe), (v, c) in expect.items():
        ov, oc = m.bellman_step(np.array([0.0, 0, 1]), pe, mx, np.array([0, 0, 1], np.uint8))
        np.testing.assert_array_equal(ov, np.array(v))
        np.testing.assert_array_equal(oc, c)
        assert np.array_equal(bits(ov), bits(golden.get(f"paper/step/m{mx}p{pe}/values")))


def test_port_steps_match_golden(golden):
    for name in golden.models():
        v = golden.get(f"{name}/stepv")
        if v is None:
            continue
        m = Model.from_arrays("port", *golden.model(name))
        for mx, pe in [(1, 1), (1, 0), (0, 1), (0, 0)]:
            ov, oc = m.bellman_step(v, pe, mx)
            assert np.array_equal(bits(ov), bits(golden.get(f"{name}/step/m{mx}p{pe}/values"))), name
            assert np.array_equal(oc, golden.get(f"{name}/step/m{mx}p{pe}/chosen")), name


def test_columns_against_break_point_lp(golden):
    """test_omax.cpp:129-148 on the same 300 columns: O-max == LP to 1e-9,
    and the port reproduces the reference expectation bit for bit."""
    lens = golden.get("cols17/lens")
    lo, up, vals = golden.get("cols17/lower"), golden.get("cols17/upper"), golden.get("cols17/values")
    off = 0
    for i, L in enumerate(lens):
        sl = slice(off, off + L)
        rows = np.arange(L, dtype=np.int32)
        e, p = oracle.robust_expectation("port", rows, lo[sl], up[sl], vals[sl], True, with_p=True)
        o = oracle.robust_expectation("port", rows, lo[sl], up[sl], vals[sl], False)
        assert bits(e) == bits(golden.get("cols17/pess")[i])
        assert bits(o) == bits(golden.get("cols17/opt")[i])
        assert abs(e - golden.get("cols17/lp_pess")[i]) <= 1e-9 * (1 + abs(e))
        assert abs(o - golden.get("cols17/lp_opt")[i]) <= 1e-9 * (1 + abs(o))
        assert (p >= lo[sl]).all() and (p <= up[sl]).all() and abs(p.sum() - 1) <= 1e-12
        assert e <= o + 1e-12
        off += L


def test_port_rejects_infeasible_column_like_reference():
    lo = np.array([0.6, 0.6])
    up = np.array([0.7, 0.7])
    with pytest.raises(oracle.OracleError) as ei:
        oracle.robust_expectation("port", np.arange(2, dtype=np.int32), lo, up, np.zeros(2), True)
    assert ei.value.kind == "ModelError"
    assert "lower bounds sum to 1.2 > 1" in ei.value.message
