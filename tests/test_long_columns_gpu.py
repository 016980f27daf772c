"""GPU parity of the long-column paths and the device generator.

* omax_sorted (CTA per column, bitonic sort + prefix scan + tree reduction):
  within 1e-13 of the reference per column and per step, identical
  iteration counts and values within 1e-9 at convergence (north_star bar);
* omax_long (exact argmin greedy, forced with RIMDP_LONG=exact): bit-exact;
* rimdp_model_generate: bit-identical to the host generator.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2401_04068_b200 import engine, problems as P

pytestmark = pytest.mark.gpu

COL_TOL = 1e-13      # one column / one step (north_star: 1e-12 per iteration)
CONV_TOL = 1e-9      # at convergence (north_star)


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def f32_ulps(q, ref):
    """Distance of float32 results from the reference, in units of the reference's last place."""
    ref = np.asarray(ref, np.float32)
    return np.abs(np.asarray(q, np.float64) - ref.astype(np.float64)) / np.spacing(np.abs(ref)).astype(np.float64)


# tree-order float32 sums (RIMDP_F32_FAST / RIMDP_LONG=select) against the reference's sequential ones over
# columns of up to 8192 entries: both carry rounding error of up to ~L/2 * 2^-24 relative (the reference's
# sequential sum is the less accurate one); measured at most 57 ulps here
F32_TREE_ULPS = 128


def with_env(name, value, fn):
    old = os.environ.get(name)
    os.environ[name] = value
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old


def with_long_mode(mode, fn):
    old = os.environ.get("RIMDP_LONG")
    os.environ["RIMDP_LONG"] = mode
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["RIMDP_LONG"]
        else:
            os.environ["RIMDP_LONG"] = old


@pytest.fixture(scope="module")
def powerlaw():
    # lengths 1 .. 8192 (every sorted size class), many greedy picks per column
    cfg = engine.gen_config(9000, 1, law=1, alpha=0.9, kmax=8192, seed=21)
    return engine.generate_host(cfg)


def tricky_values(n, seed):
    """Heavy ties (value levels), exact zeros, and near-ties that differ only in
    the low mantissa bits (exercises the truncated-key fix-up)."""
    rng = np.random.default_rng(seed)
    v = rng.integers(0, 40, n) / 40.0
    near = rng.random(n) < 0.2
    v[near] = 0.5 + rng.integers(0, 3, near.sum()) * 2.0 ** -48
    v[rng.random(n) < 0.05] = 0.0
    return v


def ref_columns(arrays, v, pess):
    sp, cp, rv, lo, up = arrays
    return np.array([oracle.robust_expectation("ref", rv[cp[c]:cp[c + 1]], lo[cp[c]:cp[c + 1]],
                                               up[cp[c]:cp[c + 1]], v, pess) for c in range(len(cp) - 1)])


def test_scheduler_routes_power_law_columns_to_the_sorted_path(powerlaw):
    m = engine.DeviceModel.from_csc(*powerlaw)
    info = m.info()
    assert info.long_columns > 100 and info.max_column_length > 4096
    assert info.short_columns + info.mid_columns + info.long_columns == m.num_cols


@pytest.mark.parametrize("mode", ["default", "select", "sorted"])
@pytest.mark.parametrize("pess", [True, False])
def test_sorted_columns_within_tolerance(powerlaw, pess, mode):
    """default: many-pick columns on the quickselect kernels; select: every
    long column there (few-pick ones too); sorted: every long column on the
    bitonic-sort kernel."""
    v = tricky_values(9000, 3)
    ref = ref_columns(powerlaw, v, pess)
    make = (lambda: engine.DeviceModel.from_csc(*powerlaw))
    m = make() if mode == "default" else with_long_mode(mode, make)
    q = m.column_values(v, pess)
    err = np.abs(q - ref)
    assert err.max() <= COL_TOL, (err.max(), int(err.argmax()), int(np.diff(powerlaw[1])[err.argmax()]))
    # deterministic: a second model gives the same bits
    m2 = make() if mode == "default" else with_long_mode(mode, make)
    assert np.array_equal(bits(q), bits(m2.column_values(v, pess)))


@pytest.mark.parametrize("pess", [True, False])
def test_select_random_values_within_tolerance(powerlaw, pess):
    """Continuous values (no ties) and the f32 store of the same columns."""
    v = np.random.default_rng(8).random(9000)
    ref = ref_columns(powerlaw, v, pess)
    q = with_long_mode("select", lambda: engine.DeviceModel.from_csc(*powerlaw)).column_values(v, pess)
    assert np.abs(q - ref).max() <= COL_TOL
    sp, cp, rv, lo, up = powerlaw
    arr32 = (sp, cp, rv, lo.astype(np.float32), up.astype(np.float32))
    v32 = v.astype(np.float32)
    ref32 = ref_columns(arr32, v32, pess)
    q32 = with_long_mode("select", lambda: engine.DeviceModel.from_csc(*arr32)).column_values(v32, pess)
    assert f32_ulps(q32, ref32).max() <= F32_TREE_ULPS


@pytest.mark.parametrize("pess", [True, False])
def test_default_random_values_within_tolerance(powerlaw, pess):
    """Default routing on continuous values, deterministic.  float64: value buckets (omax_bucket for > 256
    entries, omax_wbucket for 33-256), within 1e-13.  float32: the exact route (exact_warp / exact_sort +
    exact_dot), bit-identical; with RIMDP_F32_FAST=1 the value buckets, within a few ulps."""
    v = np.random.default_rng(9).random(9000)
    ref = ref_columns(powerlaw, v, pess)
    m = engine.DeviceModel.from_csc(*powerlaw)
    q = m.column_values(v, pess)
    assert np.abs(q - ref).max() <= COL_TOL
    assert np.array_equal(bits(q), bits(m.column_values(v, pess)))
    sp, cp, rv, lo, up = powerlaw
    arr32 = (sp, cp, rv, lo.astype(np.float32), up.astype(np.float32))
    v32 = v.astype(np.float32)
    ref32 = ref_columns(arr32, v32, pess)
    q32 = engine.DeviceModel.from_csc(*arr32).column_values(v32, pess)
    assert np.array_equal(bits(q32), bits(ref32.astype(np.float32)))
    fast = with_env("RIMDP_F32_FAST", "1", lambda: engine.DeviceModel.from_csc(*arr32)).column_values(v32, pess)
    assert f32_ulps(fast, ref32).max() <= F32_TREE_ULPS


@pytest.mark.parametrize("pess", [True, False])
@pytest.mark.parametrize("values", ["constant", "outlier", "negative"])
def test_value_buckets_degenerate_ranges(powerlaw, pess, values):
    """The value buckets span the whole vector's range: a constant vector (zero
    span: one bucket), one huge outlier (every other value in the first
    bucket) and negative values must still give the reference's columns
    (brackets too wide go to the selection fallback)."""
    rng = np.random.default_rng(12)
    if values == "constant":
        v = np.full(9000, 0.375)
    elif values == "outlier":
        v = rng.random(9000)
        v[17] = 1e6
    else:
        v = rng.random(9000) - 0.5
    ref = ref_columns(powerlaw, v, pess)
    q = engine.DeviceModel.from_csc(*powerlaw).column_values(v, pess)
    assert np.abs(q - ref).max() <= COL_TOL * max(1.0, np.abs(v).max())


@pytest.mark.parametrize("pess", [True, False])
def test_exact_long_kernel_bit_exact(powerlaw, pess):
    v = tricky_values(9000, 4)
    ref = ref_columns(powerlaw, v, pess)
    m = with_long_mode("exact", lambda: engine.DeviceModel.from_csc(*powerlaw))
    assert m.info().long_columns == 0
    assert np.array_equal(bits(m.column_values(v, pess)), bits(ref))


def test_sorted_bellman_steps_within_tolerance(powerlaw):
    cpu = oracle.Model.from_arrays("ref", *powerlaw)
    m = with_long_mode("sorted", lambda: engine.DeviceModel.from_csc(*powerlaw))
    v = tricky_values(9000, 5)
    for pess in (True, False):
        for maxi in (True, False):
            gv, gc = m.bellman_step(v, pess, maxi)
            cv, cc = cpu.bellman_step(v, pess, maxi)
            assert np.abs(gv - cv).max() <= COL_TOL


@pytest.fixture(scope="module")
def c5_small():
    """Config 5's law scaled down (4000 states x 3 actions, k <= 2048)."""
    return engine.generate_host(engine.gen_config(4000, 3, law=1, alpha=1.5, kmax=2048, seed=5))


@pytest.mark.parametrize("pess,maxi", [(True, True), (False, False), (True, False)])
def test_discounted_reward_synthesis_matches_reference(c5_small, pess, maxi):
    sp, cp, rv, lo, up = c5_small
    n = len(sp) - 1
    rng = np.random.default_rng(9)
    r = rng.random(n)
    cpu = oracle.Model.from_arrays("ref", *c5_small)
    ref = cpu.solve(oracle.Problem(oracle.INFINITE_REWARD, rewards=r, discount=0.95, eps=1e-6, pessimistic=pess,
                                   maximize=maxi), synthesize=True)
    m = engine.DeviceModel.from_csc(*c5_small)
    spec = P.Specification(P.InfiniteTimeReward(r, 0.95, 1e-6), P.PESSIMISTIC if pess else P.OPTIMISTIC,
                           P.MAXIMIZE if maxi else P.MINIMIZE)
    pol, vf = P.control_synthesis(m, spec, sp)
    assert vf.iterations == ref["iterations"]
    assert np.abs(vf.values - ref["values"]).max() <= CONV_TOL
    # strategies equal wherever the action gap exceeds the tolerance
    q = m.column_values(vf.values, pess)
    diff = np.nonzero(pol.columns != ref["policy"])[0]
    for s in diff:
        assert abs(q[pol.columns[s]] - q[ref["policy"][s]]) <= CONV_TOL, s


def test_reachability_matches_reference(c5_small):
    sp = c5_small[0]
    n = len(sp) - 1
    goal = list(range(n - 40, n))
    cpu = oracle.Model.from_arrays("ref", *c5_small)
    ref = cpu.solve(oracle.Problem(oracle.INFINITE_REACH, reach=goal, eps=1e-6))
    m = engine.DeviceModel.from_csc(*c5_small)
    vf = P.value_iteration(m, P.Specification(P.InfiniteTimeReachability(goal, 1e-6)))
    assert vf.iterations == ref["iterations"]
    assert np.abs(vf.values - ref["values"]).max() <= CONV_TOL


@pytest.mark.parametrize("law,dtype", [(0, np.float64), (1, np.float64), (1, np.float32)])
def test_device_generator_matches_host(law, dtype):
    for sb, se in ((0, 0), (700, 1500)):
        cfg = engine.gen_config(2000, 4, law=law, support=48, kmax=1500, seed=13, dtype=dtype, state_begin=sb,
                                state_end=se)
        host = engine.generate_host(cfg)
        m = engine.DeviceModel.generate(cfg)
        assert m.num_cols == len(host[1]) - 1 and m.nnz == host[1][-1]
        cp, rv, lo, gp = m.read_columns(0, m.num_cols)
        assert np.array_equal(cp, host[1])
        assert np.array_equal(rv, host[2])
        assert np.array_equal(bits(lo), bits(host[3]))
        assert np.array_equal(bits(gp), bits((host[4] - host[3]).astype(dtype)))


def test_generated_shard_steps_match_whole_model():
    """A shard computes exactly the rows of its states (the multi-GPU contract)."""
    cfg = engine.gen_config(3000, 4, law=1, kmax=512, seed=17)
    whole = engine.DeviceModel.generate(cfg)
    v = np.random.default_rng(1).random(3000)
    wv, wc = whole.bellman_step(v, True, True)
    for sb, se in ((0, 1000), (1000, 3000)):
        part = engine.DeviceModel.generate(engine.gen_config(3000, 4, law=1, kmax=512, seed=17, state_begin=sb,
                                                             state_end=se))
        pv, pc = part.bellman_step(v, True, True)
        assert np.array_equal(bits(pv[sb:se]), bits(wv[sb:se]))
        assert np.array_equal(pc + sb * 4, wc[sb:se])


@pytest.fixture(scope="module")
def fewpick():
    # C3's law at a smaller size: every column has all 400 states as support, few greedy picks
    return engine.random_imdp(400, 3, 1.0, 1.0 / 400, seed=5)


@pytest.mark.parametrize("pess", [True, False])
@pytest.mark.parametrize("values", ["tricky", "random"])
def test_single_pass_long_kernel_within_tolerance(fewpick, pess, values):
    """omax_long_tree (default for few-pick long columns): exact picks, tree-order
    sums within 1e-13 of the reference; deterministic; RIMDP_LONG=exact stays
    bit-exact on the same columns."""
    v = tricky_values(400, 6) if values == "tricky" else np.random.default_rng(9).random(400)
    ref = ref_columns(fewpick, v, pess)
    m = engine.DeviceModel.from_csc(*fewpick)
    assert m.info().mid_columns == m.num_cols  # every column on the few-pick long path
    q = m.column_values(v, pess)
    assert np.abs(q - ref).max() <= COL_TOL
    assert np.array_equal(bits(q), bits(engine.DeviceModel.from_csc(*fewpick).column_values(v, pess)))
    ex = with_long_mode("exact", lambda: engine.DeviceModel.from_csc(*fewpick))
    assert np.array_equal(bits(ex.column_values(v, pess)), bits(ref))


@pytest.mark.parametrize("pess", [True, False])
def test_single_pass_long_kernel_f32(fewpick, pess):
    """The f32 store of the same few-pick columns: the default float32 route is row-order (omax_long),
    bit-identical; the tree-order kernel (RIMDP_F32_FAST=1) within a few ulps."""
    sp, cp, rv, lo, up = fewpick
    arr32 = (sp, cp, rv, lo.astype(np.float32), up.astype(np.float32))
    v32 = np.random.default_rng(10).random(400).astype(np.float32)
    ref32 = ref_columns(arr32, v32, pess)
    q32 = engine.DeviceModel.from_csc(*arr32).column_values(v32, pess)
    assert np.array_equal(bits(q32), bits(ref32.astype(np.float32)))
    fast = with_env("RIMDP_F32_FAST", "1", lambda: engine.DeviceModel.from_csc(*arr32)).column_values(v32, pess)
    assert f32_ulps(fast, ref32).max() <= F32_TREE_ULPS
    ex = with_long_mode("exact", lambda: engine.DeviceModel.from_csc(*arr32))
    assert np.array_equal(bits(ex.column_values(v32, pess)), bits(ref32.astype(np.float32)))
