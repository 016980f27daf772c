import os, sys, numpy as np
sys.path.insert(0, ".")
from paper_2401_04068_b200 import engine
world = int(sys.argv[1]); dt = np.float32 if sys.argv[2] == "f32" else np.float64; which = int(sys.argv[3])
arrays = engine.generate_host(engine.gen_config(3000, 4, law=1, kmax=2048, seed=5, dtype=dt))
n = 3000
goal = np.zeros(n, np.uint8); goal[-10:] = 1
rew = np.random.default_rng(2).random(n).astype(dt)
g = goal.astype(dt)
plans = [dict(initial=g, frozen=goal, finite=False, eps=1e-6, pessimistic=True, maximize=True),
         dict(initial=g, frozen=goal, finite=True, horizon=17, pessimistic=False, maximize=False),
         dict(initial=rew, rewards=rew, discount=0.95, finite=False, eps=1e-6, pessimistic=True, maximize=False)]
plan = plans[which]
rec = sys.argv[4] if len(sys.argv) > 4 else "last"
m = engine.DeviceModel.from_csc(*arrays) if world == 0 else engine.MultiModel(*arrays, world=world, devices=[0] * world)
try:
    b = m.solve(record=rec, **plan)
    print(sys.argv[1:], "ok", b["iterations"], flush=True)
except Exception as e:
    print(sys.argv[1:], "FAIL", str(e)[:300], flush=True)
if len(sys.argv) > 5 and sys.argv[5] == "seq":
    for i, pl in enumerate(plans):
        try:
            b = m.solve(record=rec, **pl)
            print("seq", i, "ok", b["iterations"], flush=True)
        except Exception as e:
            print("seq", i, "FAIL", str(e)[:200], flush=True)
            break
