"""GPU parity of omax_medium: columns of 33..128 entries whose greedy needs few
picks (config 4's 64-successor columns are this class), E = 2 and 4 entries
per lane.  Bit-exact against the reference per column, per step and per
trajectory (same iteration count, same bits, same strategy)."""
import numpy as np
import pytest

import oracle
from paper_2401_04068_b200 import engine, problems as P

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def medium_model(n, actions, seed, dtype=np.float64, kmin=1, kmax=128):
    """Random columns with lengths kmin..kmax (mostly 33..128), large gaps so
    the greedy stops after a few picks, some clipped exactly at the remainder."""
    rng = np.random.default_rng(seed)
    cols, rows, lo, up = [0], [], [], []
    for c in range(n * actions):
        k = int(rng.integers(kmin, kmax + 1))
        r = np.sort(rng.choice(n, k, replace=False))
        l = rng.random(k) * (0.6 / k)
        u = np.minimum(l + rng.random(k), 1.0)
        if c % 7 == 0:  # a few degenerate entries (u == l) and zero lower bounds
            l[::5] = 0.0
            u[1::6] = l[1::6]
            u[0] = 1.0
        if u.sum() < 1:
            u[:] = 1.0
        rows += list(r)
        lo += list(l)
        up += list(u)
        cols.append(len(rows))
    sp = np.arange(0, n * actions + 1, actions, dtype=np.int32)
    return (sp, np.array(cols, np.int64), np.array(rows, np.int32), np.array(lo, dtype), np.array(up, dtype))


def values(n, seed, dtype=np.float64):
    rng = np.random.default_rng(seed)
    v = rng.integers(0, 25, n) / 25.0        # heavy ties: position order decides
    cont = rng.random(n) < 0.3
    v[cont] = rng.random(cont.sum())
    v[rng.random(n) < 0.05] = 0.0
    return v.astype(dtype)


@pytest.fixture(scope="module", params=[np.float64, np.float32], ids=["f64", "f32"])
def model(request):
    return medium_model(1500, 3, 11, request.param)


@pytest.mark.parametrize("pess", [True, False])
def test_medium_columns_bit_exact(model, pess):
    dtype = model[3].dtype
    v = values(1500, 2, dtype)
    sp, cp, rv, lo, up = model
    ref = np.array([oracle.robust_expectation("ref", rv[cp[c]:cp[c + 1]], lo[cp[c]:cp[c + 1]], up[cp[c]:cp[c + 1]],
                                              v, pess) for c in range(len(cp) - 1)], dtype)
    m = engine.DeviceModel.from_csc(*model)
    info = m.info()
    assert info.mid_columns > 1000 and info.max_column_length > 64
    q = m.column_values(v, pess)
    bad = np.flatnonzero(bits(q) != bits(ref))
    assert bad.size == 0, (bad[:5], q[bad[:5]], ref[bad[:5]], np.diff(cp)[bad[:5]])


def test_medium_bellman_steps_bit_exact(model):
    dtype = model[3].dtype
    cpu = oracle.Model.from_arrays("ref", *model)
    m = engine.DeviceModel.from_csc(*model)
    v = values(1500, 3, dtype)
    frozen = (np.arange(1500) % 13 == 0).astype(np.uint8)
    for pess in (True, False):
        for maxi in (True, False):
            gv, gc = m.bellman_step(v, pess, maxi, frozen)
            cv, cc = cpu.bellman_step(v, pess, maxi, frozen)
            assert np.array_equal(bits(gv), bits(cv))
            assert np.array_equal(gc, cc)


def test_c4_shape_solve_bit_exact():
    """Config 4's law (64 stratified successors, lower = u/64) scaled to 5000
    states x 8 actions: the full Pmaxmin reachability solve."""
    n = 5000
    cfg = engine.gen_config(n, 8, law=0, support=64, seed=1)
    arrays = engine.generate_host(cfg)
    goal = np.zeros(n, np.uint8)
    goal[-n // 100:] = 1
    m = engine.DeviceModel.from_csc(*arrays)
    assert m.info().mid_columns == 8 * n
    cpu = oracle.Model.from_arrays("ref", *arrays)
    spec = P.Specification(P.InfiniteTimeReachability(list(np.flatnonzero(goal)), 1e-6))
    pol, vf = P.control_synthesis(m, spec, arrays[0])
    ref = cpu.solve(oracle.Problem(oracle.INFINITE_REACH, reach=list(np.flatnonzero(goal)), eps=1e-6),
                    synthesize=True)
    assert vf.iterations == ref["iterations"]
    assert np.array_equal(bits(vf.values), bits(ref["values"]))
    assert np.array_equal(pol.columns, ref["policy"])
