"""Where the end-to-end solve loop spends time beyond the kernels (C2): a finite-horizon solve of the
same number of iterations (no stop test) against the infinite-horizon solve, both through the public
call, with RIMDP_TRACE phase times on stderr."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_04068_b200 import engine  # noqa: E402

arr = engine.random_imdp(100000, 4, 32.0 / 100000, 1.0 / 32, 1)
n = 100000
goal = np.zeros(n, np.uint8)
goal[-1000:] = 1
m = engine.DeviceModel.from_csc(*arr)
for rep in range(3):
    for finite in (False, True):
        kw = dict(initial=goal.astype(np.float64), frozen=goal, pessimistic=True, maximize=True)
        kw.update(dict(finite=True, horizon=1123) if finite else dict(finite=False, eps=1e-6))
        t = time.perf_counter()
        r = m.solve(**kw)
        dt = time.perf_counter() - t
        print(f"finite={finite} iterations={r['iterations']} {1e3 * dt:.2f} ms "
              f"({1e3 * dt / r['iterations']:.4f} ms/it)", flush=True)
