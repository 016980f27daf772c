"""The engine's workload generator reproduces the reference generator's models
byte for byte (random_model.hpp:42-161), so GPU and CPU runs ingest identical
inputs.  The expected arrays are golden fixtures exported from the reference."""
import numpy as np
import pytest

from paper_2401_04068_b200 import engine

CASES = {
    "r15s1": dict(states=15, actions=3, density=0.3, scale=0.2, seed=1),
    "r10s10": dict(states=10, actions=2, density=0.4, scale=0.2, seed=10),
    "r12s77": dict(states=12, actions=2, density=0.5, scale=0.2, seed=77),
    "pt12s21": dict(states=12, actions=3, density=0.4, scale=0.2, seed=21, point=True),
    "r200l": dict(states=200, actions=3, density=0.3, scale=1.0 / 60, seed=5),
    "r120d": dict(states=120, actions=2, density=1.0, scale=1.0 / 120, seed=6),
    "r400m": dict(states=400, actions=4, density=24.0 / 400, scale=1.0 / 24, seed=8),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_random_imdp_matches_reference_generator(golden, name):
    got = engine.random_imdp(**CASES[name])
    for g, e in zip(got, golden.model(name)):
        assert np.array_equal(np.asarray(g), np.asarray(e).astype(np.asarray(g).dtype)), name
        if np.asarray(g).dtype.kind == "f":
            assert np.array_equal(np.asarray(g).view(np.uint64), np.asarray(e).view(np.uint64))


def test_random_imdp_f32_matches_reference_generator(golden):
    got = engine.random_imdp(60, 3, 0.2, 1.0 / 12, 9, dtype=np.float32)
    for g, e in zip(got, golden.model("f32r60")):
        assert np.array_equal(np.asarray(g), np.asarray(e))


def test_bench_weak_scaling_keeps_per_gpu_work():
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    c2 = bench.WORKLOADS["c2"]
    w1, k1 = bench.scaled_workload(c2, 1, "weak")
    w8, k8 = bench.scaled_workload(c2, 8, "weak")
    assert w1 is c2 and k1 == "weak" and k8 == "weak"
    # N x the states, 32 successors per column from the counter generator (each rank builds its shard in HBM)
    assert w8["states"] == 8 * c2["states"] and w8["source"] == "generated" and w8["law"] == 0
    assert w8["support"] == 32 and w8["actions"] == c2["actions"]
    w4, k4 = bench.scaled_workload(bench.WORKLOADS["c4"], 4, "weak")
    assert w4["states"] == bench.WORKLOADS["c4"]["states"] and k4 == "strong"
    ws, ks = bench.scaled_workload(c2, 8, "strong")
    assert ws is c2 and ks == "strong"
