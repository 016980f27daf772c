set -x
ldd paper_2401_04068_b200/lib/librimdp_b200.so
ls -la --time-style=full-iso paper_2401_04068_b200/lib/ paper_2401_04068_b200/csrc/ | head -20
cat > /tmp/dbg.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2401_04068_b200 import engine
print("count", engine.device_count(), flush=True)
sp = np.array([0, 2, 4, 5], np.int32)
cp = np.array([0, 3, 6, 9, 12, 13], np.int64)
rv = np.array([0, 1, 2] * 4 + [2], np.int32)
lo = np.array([0.0, 0.1, 0.2, 0.5, 0.3, 0.1, 0.1, 0.2, 0.3, 0.2, 0.3, 0.4, 1.0])
up = np.array([0.5, 0.6, 0.7, 0.7, 0.5, 0.3, 0.6, 0.5, 0.4, 0.6, 0.5, 0.4, 1.0])
m = engine.DeviceModel.from_csc(sp, cp, rv, lo, up)
print("created", m.info().nnz, flush=True)
v, c = m.bellman_step(np.array([0.0, 0, 1]), True, True, np.array([0,0,1], np.uint8))
print("step", v, c, flush=True)
out = m.solve(initial=np.array([0.0,0,1]), frozen=np.array([0,0,1],np.uint8), finite=True, horizon=10, record="all")
print("solve", out, flush=True)
PY
python -X faulthandler /tmp/dbg.py 2>&1 | tail -30
cuda-gdb -batch -ex run -ex bt --args python /tmp/dbg.py 2>&1 | tail -40
