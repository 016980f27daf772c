import subprocess, sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
torch.zeros(1, device="cuda")
from paper_2401_04068_b200 import engine, problems as P
n = 100000
arrays = engine.random_imdp(n, 4, 32.0 / n, 1.0 / 32, seed=1)
spec = P.Specification(P.InfiniteTimeReachability(list(range(n - n // 100, n)), 1e-6))
engine.DeviceModel.from_csc(*arrays).close()
def run(tag):
    for rep in range(4):
        t0 = time.perf_counter(); m = engine.DeviceModel.from_csc(*arrays); t1 = time.perf_counter()
        vf = P.value_iteration(m, spec); t2 = time.perf_counter(); m.close()
        print(tag, f"upload {1e3*(t1-t0):.1f} solve {1e3*(t2-t1):.1f} total {1e3*(t2-t0):.1f}", flush=True)
run("nosmi")
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown", "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.DEVNULL)
time.sleep(0.5)
run("smi")
p.terminate()
time.sleep(0.5)
run("nosmi2")
