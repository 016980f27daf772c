"""Where the end-to-end time of a host-buffer solve goes (C2 by default):
model upload (rimdp_model_create: H2D + prepare_columns + schedule), solve
(plan upload + iterations + download)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_04068_b200 import engine, problems as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
arrays = engine.random_imdp(n, 4, 32.0 / n, 1.0 / 32, seed=1)
spec = P.Specification(P.InfiniteTimeReachability(list(range(n - n // 100, n)), 1e-6))
engine.DeviceModel.from_csc(*arrays).close()  # warm (context, module load)
for rep in range(3):
    t0 = time.perf_counter()
    m = engine.DeviceModel.from_csc(*arrays)
    t1 = time.perf_counter()
    vf = P.value_iteration(m, spec)
    t2 = time.perf_counter()
    m.close()
    print(f"upload {1e3 * (t1 - t0):.1f} ms  solve {1e3 * (t2 - t1):.1f} ms ({vf.iterations} it, "
          f"{1e3 * (t2 - t1) / vf.iterations:.4f} ms/it)  total {1e3 * (t2 - t0):.1f} ms  "
          f"H2D {sum(a.nbytes for a in arrays) / 1e6:.0f} MB")
