"""GPU tests of the runtime around the kernels: programmatic dependent launch
(PDL) must not change a single bit, and device memory recycled through the
stream-ordered pool must give the same results model after model."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2401_04068_b200 import engine, problems as P

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SOLVE = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
from paper_2401_04068_b200 import engine, problems as P
n = 3000
m = engine.DeviceModel.from_csc(*engine.random_imdp(n, 4, 32.0 / n, 1.0 / 32, seed=7))
vf = P.value_iteration(m, P.Specification(P.InfiniteTimeReachability(list(range(n - 30, n)), 1e-6)))
print(vf.iterations, hashlib.sha256(vf.values.tobytes() + vf.residual.tobytes()).hexdigest())
"""


def run_solve(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SOLVE.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=600, check=True)
    return out.stdout.strip().splitlines()[-1]


def test_pdl_launches_are_bit_identical_to_plain_launches():
    """C2-shaped iterations (two launches) go through launch_pdl; RIMDP_PDL=0
    launches the same kernels plainly."""
    assert run_solve({"RIMDP_PDL": "1"}) == run_solve({"RIMDP_PDL": "0"})


def test_recycled_device_memory_gives_identical_solves():
    """Models of different sizes created and destroyed back to back reuse the
    pool's memory; every solve of the same model is bit-identical."""
    n = 2000
    arrays = engine.random_imdp(n, 3, 20.0 / n, 1.0 / 20, seed=3)
    spec = P.Specification(P.InfiniteTimeReachability(list(range(n - 20, n)), 1e-6))
    ref = None
    for rep in range(6):
        no = 500 * (rep + 1)
        other = engine.DeviceModel.from_csc(*engine.random_imdp(no, 2, 10.0 / no, 0.1, seed=rep))
        m = engine.DeviceModel.from_csc(*arrays)
        vf = P.value_iteration(m, spec)
        digest = hashlib.sha256(vf.values.tobytes() + vf.residual.tobytes()).hexdigest()
        ref = ref or (vf.iterations, digest)
        assert (vf.iterations, digest) == ref
        if rep % 2:
            other.close()
        m.close()
