"""GPU parity of the tiny classes (1-4, 5-8, 9-16 entries: omax_tiny_rank, the
default, over list-ordered packed copies of the columns).  The columns are built
so the greedy takes many picks (small lower bounds, gaps of the order of rem,
some clipped exactly at the remainder) and the values carry heavy ties, so the
in-segment (key, position) ranks and the replayed `consumed` chain both
matter.  Bit-exact against the reference per column and per Bellman step."""
import numpy as np
import pytest

import oracle
from paper_2401_04068_b200 import engine

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def tiny_model(n, actions, seed, dtype):
    rng = np.random.default_rng(seed)
    cols, rows, lo, up = [0], [], [], []
    for c in range(n * actions):
        k = int(rng.integers(1, 17))
        r = np.sort(rng.choice(n, k, replace=False))
        l = rng.random(k) * (0.3 / k)
        g = rng.random(k) * (2.0 / k)
        if c % 5 == 0:
            g[::3] = 0.0                      # degenerate entries (u == l)
        u = np.minimum(l + g, 1.0)
        if u.sum() < 1:
            u[:] = 1.0
        if k == 1:
            l[:], u[:] = 0.25, 1.0
        rows += list(r)
        lo += list(l)
        up += list(u)
        cols.append(len(rows))
    sp = np.arange(0, n * actions + 1, actions, dtype=np.int32)
    return (sp, np.array(cols, np.int64), np.array(rows, np.int32), np.array(lo, dtype), np.array(up, dtype))


def tie_values(n, seed, dtype):
    rng = np.random.default_rng(seed)
    v = rng.integers(0, 6, n) / 5.0           # six distinct values: most segments hold equal keys
    cont = rng.random(n) < 0.2
    v[cont] = rng.random(cont.sum())
    v[rng.random(n) < 0.05] = -0.0            # -0 orders as +0 (ties by position)
    return v.astype(dtype)


@pytest.fixture(scope="module", params=[np.float64, np.float32], ids=["f64", "f32"])
def model(request):
    return tiny_model(4000, 3, 21, request.param)


@pytest.mark.parametrize("pess", [True, False])
def test_tiny_columns_bit_exact(model, pess):
    dtype = model[3].dtype
    sp, cp, rv, lo, up = model
    m = engine.DeviceModel.from_csc(*model)
    for seed in (1, 2):
        v = tie_values(4000, seed, dtype)
        ref = np.array([oracle.robust_expectation("ref", rv[cp[c]:cp[c + 1]], lo[cp[c]:cp[c + 1]],
                                                  up[cp[c]:cp[c + 1]], v, pess)
                        for c in range(len(cp) - 1)], dtype)
        q = m.column_values(v, pess)
        bad = np.flatnonzero(bits(q) != bits(ref))
        assert bad.size == 0, (bad[:5], q[bad[:5]], ref[bad[:5]], np.diff(cp)[bad[:5]])
    m.close()


def test_tiny_bellman_steps_bit_exact(model):
    dtype = model[3].dtype
    cpu = oracle.Model.from_arrays("ref", *model)
    m = engine.DeviceModel.from_csc(*model)
    v = tie_values(4000, 3, dtype)
    frozen = (np.arange(4000) % 11 == 0).astype(np.uint8)
    for pess in (True, False):
        for maxi in (True, False):
            gv, gc = m.bellman_step(v, pess, maxi, frozen)
            cv, cc = cpu.bellman_step(v, pess, maxi, frozen)
            assert np.array_equal(bits(gv), bits(cv))
            assert np.array_equal(gc, cc)
    m.close()
