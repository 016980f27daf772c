"""A small workload that launches every kernel family once or a few times, for compute-sanitizer
(memcheck / racecheck / synccheck): short, long, tiny, medium, bucket, wbucket, select, sorted, exact
(float32), validation, generator, multi-shard (one device, sequential: no spin across shards here)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_04068_b200 import engine  # noqa: E402


def run(arrays, dtype, label):
    n = len(arrays[0]) - 1
    rng = np.random.default_rng(1)
    m = engine.DeviceModel.from_csc(*arrays)
    for pess in (True, False):
        v = rng.random(n).astype(dtype)
        m.column_values(v, pess)
        v2 = (rng.integers(0, 4, n) / 3).astype(dtype)  # ties: bucket / exact fallbacks
        m.column_values(v2, pess)
    goal = np.zeros(n, np.uint8)
    goal[-5:] = 1
    m.solve(initial=goal.astype(dtype), frozen=goal, finite=True, horizon=6, record="all")
    r = rng.random(n).astype(dtype)
    m.solve(initial=r, rewards=r, discount=0.9, finite=False, eps=1e-3, record="last")
    m.close()
    print("ok", label, flush=True)


for dt in (np.float64, np.float32):
    run(engine.generate_host(engine.gen_config(1500, 2, law=1, alpha=0.9, kmax=8192, seed=21, dtype=dt)), dt, "power")
    run(engine.random_imdp(300, 3, 24.0 / 300, 1.0 / 24, 7, dtype=dt), dt, "short")
    run(engine.generate_host(engine.gen_config(400, 4, law=0, support=64, seed=2, dtype=dt)), dt, "medium")
    os.environ["RIMDP_LONG"] = "exact"
    run(engine.random_imdp(200, 2, 1.0, 1.0 / 200, 6, dtype=dt), dt, "long-exact")
    os.environ["RIMDP_LONG"] = "sorted"
    run(engine.generate_host(engine.gen_config(600, 2, law=1, alpha=0.9, kmax=2048, seed=3, dtype=dt)), dt, "sorted")
    del os.environ["RIMDP_LONG"]
    run(engine.random_imdp(200, 2, 1.0, 1.0 / 200, 6, dtype=dt), dt, "long-tree")
g = engine.DeviceModel.generate(engine.gen_config(2000, 4, law=1, kmax=512, seed=4))
g.close()
print("sanitize workload done")
