"""Model upload time of config 2's host arrays (RIMDP_TRACE phase 'upload'), for the staging thread count."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_04068_b200 import engine
arrays = engine.random_imdp(100000, 4, 32.0 / 100000, 1.0 / 32, 1)
for _ in range(3):
    t = time.perf_counter()
    m = engine.DeviceModel.from_csc(*arrays)
    dt = time.perf_counter() - t
    m.close()
print(os.environ.get("RIMDP_UPLOAD_THREADS", "default"), f"create {dt * 1e3:.1f} ms")
