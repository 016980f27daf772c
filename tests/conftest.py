import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a engine")
    config.addinivalue_line("markers", "slow: long-running parity case")


class Golden:
    """tests/golden/small.npz + small.json, produced by make_golden.py from the reference."""

    def __init__(self):
        self.arr = np.load(os.path.join(GOLDEN, "small.npz"))
        with open(os.path.join(GOLDEN, "small.json")) as f:
            self.meta = json.load(f)

    def model(self, name):
        a = self.arr
        return (a[f"{name}/stateptr"], a[f"{name}/colptr"], a[f"{name}/rowval"], a[f"{name}/lower"],
                a[f"{name}/upper"])

    def models(self):
        return sorted({k.split("/")[0] for k in self.arr.files if k.endswith("/stateptr")})

    def solves(self, model=None):
        return sorted(k for k, v in self.meta.items() if "kind" in v and (model is None or k.startswith(model + "/")))

    def get(self, key, default=None):
        return self.arr[key] if key in self.arr.files else default


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def engine_lib():
    """The built engine library (built in-tree on demand; never a fallback)."""
    from paper_2401_04068_b200 import build, engine
    build.build()  # no-op when the in-tree library is up to date
    return engine.load()
