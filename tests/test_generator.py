"""Counter-based workload generator (csrc/generator.cuh) on the host: the laws
of BASELINE configs 4-5, column independence (any shard
regenerates the same columns) and feasibility of every column."""
import numpy as np
import pytest

from paper_2401_04068_b200 import engine


def _check_columns(sp, cp, rv, lo, up, n):
    lens = np.diff(cp)
    assert (lens >= 1).all()
    for c in range(len(lens)):
        r = rv[cp[c]:cp[c + 1]]
        assert (np.diff(r) > 0).all() and r[0] >= 0 and r[-1] < n  # strictly increasing rows (csc.hpp:98-101)
    assert (lo >= 0).all() and (lo <= up).all() and (up <= 1).all()
    ls = np.add.reduceat(lo.astype(np.float64), cp[:-1])
    us = np.add.reduceat(up.astype(np.float64), cp[:-1])
    assert (ls <= 1 + 1e-9).all() and (us >= 1 - 1e-9).all()  # feasible (interval.hpp:132-179)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fixed_support_law(dtype):
    cfg = engine.gen_config(500, 8, law=0, support=64, seed=7, dtype=dtype)
    sp, cp, rv, lo, up = engine.generate_host(cfg)
    assert len(cp) - 1 == 4000 and cp[-1] == 4000 * 64 and list(sp[:3]) == [0, 8, 16]
    assert lo.dtype == dtype
    _check_columns(sp, cp, rv, lo, up, 500)
    # lower = u / 64: mean 1/128
    assert abs(float(lo.mean()) - 1 / 128) < 2e-4


def test_power_law_lengths():
    cfg = engine.gen_config(20000, 4, law=1, alpha=1.5, kmax=4096, seed=11)
    sp, cp, rv, lo, up = engine.generate_host(cfg)
    lens = np.diff(cp)
    _check_columns(sp, cp, rv, lo, up, 20000)
    # P(k) ~ k^-1.5 on [1, 4096]: P(k = 1) = 1 / zeta_4096(1.5) ~ 0.386, mean ~ 49.5
    k = np.arange(1, 4097, dtype=np.float64)
    w = k ** -1.5
    assert abs((lens == 1).mean() - w[0] / w.sum()) < 0.01
    assert abs(lens.mean() - (k * w).sum() / w.sum()) < 8
    assert lens.max() > 1024


@pytest.mark.parametrize("law", [0, 1])
def test_shards_regenerate_the_same_columns(law):
    full = engine.generate_host(engine.gen_config(900, 3, law=law, support=40, kmax=600, seed=5))
    for sb, se in ((0, 300), (300, 301), (301, 900)):
        part = engine.generate_host(engine.gen_config(900, 3, law=law, support=40, kmax=600, seed=5, state_begin=sb,
                                                      state_end=se))
        cb, ce = sb * 3, se * 3
        b, e = full[1][cb], full[1][ce]
        assert np.array_equal(part[1], full[1][cb:ce + 1] - b)
        for x, y in zip(part[2:], full[2:]):
            assert np.array_equal(x, y[b:e])


def test_seed_changes_the_model():
    a = engine.generate_host(engine.gen_config(100, 2, law=1, kmax=64, seed=1))
    b = engine.generate_host(engine.gen_config(100, 2, law=1, kmax=64, seed=2))
    assert not (len(a[2]) == len(b[2]) and np.array_equal(a[2], b[2]))


def test_invalid_configs_rejected():
    with pytest.raises(engine.EngineError):
        engine.generate_host(engine.gen_config(100, 2, law=1, kmax=100000))
    with pytest.raises(engine.EngineError):
        engine.generate_host(engine.gen_config(100, 2, law=0, state_begin=50, state_end=20))
