"""Generate the golden fixtures in tests/golden from the reference itself.

Run in the dev container (needs /root/reference and oracle/_ref):

    python tests/golden/make_golden.py            # small fixtures
    python tests/golden/make_golden.py --c2 --c3  # config-2/3 convergence digests (minutes)
    python tests/golden/make_golden.py --c5s      # config-5 law at 30000 states, f64 + f32 (a minute)

Every number comes from the unmodified reference headers compiled by
oracle/Makefile (oracle/_ref/librimdp_ref.so): random_imdp / random_point_imdp
(random_model.hpp), value_iteration / control_synthesis / verify_policy
(solver.hpp), bellman_step (bellman.hpp), robust_expectation (omax.hpp) and
the reference tests' break-point LP (tests/oracle.hpp).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import Model, Problem  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MODES = [(1, 1), (1, 0), (0, 1), (0, 0)]  # (maximize, pessimistic)


def paper_arrays():
    """The §3.1 model (reference test_solver.cpp:13-25), aligned CSC."""
    lo = [[0.0, 0.1, 0.2], [0.5, 0.3, 0.1], [0.1, 0.2, 0.3], [0.2, 0.3, 0.4], [0, 0, 1.0]]
    up = [[0.5, 0.6, 0.7], [0.7, 0.5, 0.3], [0.6, 0.5, 0.4], [0.6, 0.5, 0.4], [0, 0, 1.0]]
    cp, rv, L, U = [0], [], [], []
    for lcol, ucol in zip(lo, up):
        for r in range(3):
            if lcol[r] != 0 or ucol[r] != 0:
                rv.append(r)
                L.append(lcol[r])
                U.append(ucol[r])
        cp.append(len(rv))
    return (np.array([0, 2, 4, 5], np.int32), np.array(cp, np.int64), np.array(rv, np.int32),
            np.array(L), np.array(U))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def solve_record(m: Model, pr: Problem, synth=True, trace=0):
    try:
        out = m.solve(pr, synthesize=synth, trace_iters=trace)
        return {"ok": True, **out}
    except oracle.OracleError as e:
        return {"ok": False, "kind": e.kind, "message": e.message, "iterations": e.iterations}


def add_model(store, name, arrays):
    sp, cp, rv, lo, up = arrays
    store[f"{name}/stateptr"] = sp
    store[f"{name}/colptr"] = cp
    store[f"{name}/rowval"] = rv
    store[f"{name}/lower"] = lo
    store[f"{name}/upper"] = up


def add_solve(store, meta, key, res, pr: Problem):
    meta[key] = {"kind": pr.kind, "reach": list(map(int, pr.reach)), "avoid": list(map(int, pr.avoid)),
                 "horizon": int(pr.horizon), "eps": pr.eps, "pessimistic": int(pr.pessimistic),
                 "maximize": int(pr.maximize), "discount": pr.discount, "max_iterations": pr.max_iterations,
                 "ok": res["ok"]}
    if pr.rewards is not None:
        store[f"{key}/rewards"] = np.asarray(pr.rewards)
    if res["ok"]:
        store[f"{key}/values"] = res["values"]
        store[f"{key}/residual"] = res["residual"]
        meta[key]["iterations"] = int(res["iterations"])
        if "policy" in res:
            store[f"{key}/policy"] = res["policy"]
        if "trace" in res:
            store[f"{key}/trace"] = res["trace"]
    else:
        meta[key].update({"error": res["kind"], "message": res["message"], "iterations": res["iterations"]})


def small():
    store: dict = {}
    meta: dict = {}
    # ---- the paper model, all modes --------------------
    arrays = paper_arrays()
    add_model(store, "paper", arrays)
    m = Model.from_arrays("ref", *arrays)
    for mx, pe in MODES:
        for kind, kw in ((oracle.FINITE_REACH, {"horizon": 10}), (oracle.FINITE_REACH, {"horizon": 100}),
                         (oracle.INFINITE_REACH, {"eps": 1e-6}), (oracle.INFINITE_REACH, {"eps": 1e-8})):
            pr = Problem(kind, reach=[2], pessimistic=pe, maximize=mx, **kw)
            tag = f"h{kw['horizon']}" if "horizon" in kw else f"e{kw['eps']:g}"
            add_solve(store, meta, f"paper/{tag}/m{mx}p{pe}", solve_record(m, pr, trace=100), pr)
        v, c = m.bellman_step(np.array([0.0, 0, 1]), pe, mx, np.array([0, 0, 1], np.uint8))
        store[f"paper/step/m{mx}p{pe}/values"] = v
        store[f"paper/step/m{mx}p{pe}/chosen"] = c
    for h in (0, 1, 100):
        pr = Problem(oracle.FINITE_REWARD, rewards=np.array([1.0, 2.0, 3.0]), discount=0.95, horizon=h)
        add_solve(store, meta, f"paper/reward_h{h}", solve_record(m, pr), pr)
    pr = Problem(oracle.INFINITE_REWARD, rewards=np.array([1.0, 2.0, 3.0]), discount=0.9, eps=1e-10)
    add_solve(store, meta, "paper/reward_inf", solve_record(m, pr), pr)
    pr = Problem(oracle.INFINITE_REACH, reach=[2], eps=1e-300, max_iterations=2)
    add_solve(store, meta, "paper/nonconv", solve_record(m, pr, synth=False), pr)

    # ---- random models from the reference generator ------------------------
    specs = [
        ("r15s1", dict(states=15, actions=3, density=0.3, scale=0.2, seed=1)),
        ("r15s2", dict(states=15, actions=3, density=0.3, scale=0.2, seed=2)),
        ("r10s10", dict(states=10, actions=2, density=0.4, scale=0.2, seed=10)),
        ("r10s11", dict(states=10, actions=2, density=0.4, scale=0.2, seed=11)),
        ("r12s77", dict(states=12, actions=2, density=0.5, scale=0.2, seed=77)),
        ("r14s41", dict(states=14, actions=3, density=0.3, scale=0.2, seed=41)),
        ("pt12s21", dict(states=12, actions=3, density=0.4, scale=0.2, seed=21, point=True)),
        # long-column shapes (> 32 successors) for the long path
        ("r200l", dict(states=200, actions=3, density=0.3, scale=1.0 / 60, seed=5)),
        ("r120d", dict(states=120, actions=2, density=1.0, scale=1.0 / 120, seed=6)),
        ("r400m", dict(states=400, actions=4, density=24.0 / 400, scale=1.0 / 24, seed=8)),
    ]
    for name, kw in specs:
        point = kw.pop("point", False)
        rm = Model.random(**kw, point=point)
        arrays = rm.export()
        add_model(store, name, arrays)
        n = kw["states"]
        goal = [n - 1]
        for mx, pe in MODES:
            pr = Problem(oracle.FINITE_REACH, reach=goal, horizon=30, pessimistic=pe, maximize=mx)
            add_solve(store, meta, f"{name}/h30/m{mx}p{pe}", solve_record(rm, pr, trace=30), pr)
            pr = Problem(oracle.INFINITE_REACH, reach=goal, eps=1e-6, pessimistic=pe, maximize=mx,
                         max_iterations=5000)
            add_solve(store, meta, f"{name}/e1e-06/m{mx}p{pe}", solve_record(rm, pr), pr)
        # reach-avoid and reward on every model
        pr = Problem(oracle.FINITE_REACH_AVOID, reach=[n - 1], avoid=[0, 1], horizon=40)
        add_solve(store, meta, f"{name}/ra40", solve_record(rm, pr), pr)
        pr = Problem(oracle.INFINITE_REACH_AVOID, reach=[n - 1], avoid=[0, 1], eps=1e-7, max_iterations=5000)
        add_solve(store, meta, f"{name}/ra_inf", solve_record(rm, pr), pr)
        rew = (np.arange(n) % 7) / 7.0
        pr = Problem(oracle.INFINITE_REWARD, rewards=rew, discount=0.95, eps=1e-6)
        add_solve(store, meta, f"{name}/rew_inf", solve_record(rm, pr), pr)
        # verify the synthesized stationary policy (solver.hpp:204-251)
        pr = Problem(oracle.INFINITE_REACH, reach=goal, eps=1e-6, max_iterations=5000)
        syn = solve_record(rm, pr)
        if syn["ok"]:
            ver = rm.verify_policy(pr, syn["policy"])
            store[f"{name}/verify/policy"] = syn["policy"]
            store[f"{name}/verify/values"] = ver["values"]
            meta[f"{name}/verify"] = {"iterations": int(ver["iterations"])}
        # one Bellman step from a random V, both directions
        rng = np.random.default_rng(3)
        v = rng.random(n)
        v[::5] = v[1::5][: len(v[::5])] if n > 5 else v[::5]  # ties
        store[f"{name}/stepv"] = v
        for mx, pe in MODES:
            ov, oc = rm.bellman_step(v, pe, mx)
            store[f"{name}/step/m{mx}p{pe}/values"] = ov
            store[f"{name}/step/m{mx}p{pe}/chosen"] = oc

    # ---- f32 instantiation ---------------------------------------------------
    rm = Model.random(states=60, actions=3, density=0.2, scale=1.0 / 12, seed=9, dtype=np.float32)
    add_model(store, "f32r60", rm.export())
    for mx, pe in MODES:
        pr = Problem(oracle.FINITE_REACH, reach=[59], horizon=25, pessimistic=pe, maximize=mx)
        add_solve(store, meta, f"f32r60/h25/m{mx}p{pe}", solve_record(rm, pr), pr)
    pr = Problem(oracle.INFINITE_REWARD, rewards=(np.arange(60) % 5 / 5.0).astype(np.float32), discount=0.95,
                 eps=1e-5)
    add_solve(store, meta, "f32r60/rew_inf", solve_record(rm, pr), pr)

    # ---- columns of the reference tests (test_omax.cpp:73-208) -----------------
    lens, lo, up, vals = oracle.test_columns(17, 300)
    store["cols17/lens"] = lens
    store["cols17/lower"] = lo
    store["cols17/upper"] = up
    store["cols17/values"] = vals
    exp_p, exp_o, lp_p, lp_o, pp = [], [], [], [], []
    off = 0
    for L in lens:
        sl = slice(off, off + L)
        rows = np.arange(L, dtype=np.int32)
        e, p = oracle.robust_expectation("ref", rows, lo[sl], up[sl], vals[sl], True, with_p=True)
        exp_p.append(e)
        pp.append(p)
        exp_o.append(oracle.robust_expectation("ref", rows, lo[sl], up[sl], vals[sl], False))
        lp_p.append(oracle.lp_expectation(lo[sl], up[sl], vals[sl], True))
        lp_o.append(oracle.lp_expectation(lo[sl], up[sl], vals[sl], False))
        off += L
    store["cols17/pess"] = np.array(exp_p)
    store["cols17/opt"] = np.array(exp_o)
    store["cols17/lp_pess"] = np.array(lp_p)
    store["cols17/lp_opt"] = np.array(lp_o)
    store["cols17/p_pess"] = np.concatenate(pp)

    np.savez_compressed(os.path.join(OUT, "small.npz"), **store)
    with open(os.path.join(OUT, "small.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote small.npz", len(store), "arrays;", len(meta), "solves")


def big(which: str):
    """Convergence digests of BASELINE configs 2/3, ref, all threads."""
    import time
    if which == "c2":
        cfg = dict(states=100000, actions=4, density=32.0 / 100000, scale=1.0 / 32, seed=1)
        goal = list(range(99000, 100000))
        modes = [(1, 1)]
    else:
        cfg = dict(states=2000, actions=10, density=1.0, scale=1.0 / 2000, seed=1)
        goal = list(range(1980, 2000))
        modes = [(0, 1), (1, 1)]
    rm = Model.random(**cfg)
    res = {"config": cfg, "goal": [goal[0], goal[-1] + 1], "runs": {}}
    full = {}
    for mx, pe in modes:
        pr = Problem(oracle.INFINITE_REACH, reach=goal, eps=1e-6, pessimistic=pe, maximize=mx)
        t = time.time()
        out = rm.solve(pr, synthesize=True)
        dt = time.time() - t
        v = out["values"]
        res["runs"][f"m{mx}p{pe}"] = {
            "iterations": int(out["iterations"]), "seconds": dt, "threads": os.cpu_count(),
            "values_sha256": digest(v), "residual_sha256": digest(out["residual"]),
            "policy_sha256": digest(out["policy"].astype(np.int32)),
            "vmin": float(v.min()), "vmax": float(v.max()), "max_residual": float(out["residual"].max()),
            "sample_idx": list(range(0, cfg["states"], cfg["states"] // 16)),
            "sample_hex": [float(v[i]).hex() for i in range(0, cfg["states"], cfg["states"] // 16)],
        }
        print(which, mx, pe, res["runs"][f"m{mx}p{pe}"]["iterations"], f"{dt:.1f}s", flush=True)
        if which == "c3":  # 2000 states: the whole vectors are small enough to keep
            full[f"m{mx}p{pe}/values"] = v
            full[f"m{mx}p{pe}/residual"] = out["residual"]
            full[f"m{mx}p{pe}/policy"] = out["policy"].astype(np.int32)
    with open(os.path.join(OUT, f"{which}.json"), "w") as f:
        json.dump(res, f, indent=1)
    if full:
        np.savez_compressed(os.path.join(OUT, f"{which}_full.npz"), **full)


def c5_scaled(states=30000):
    """BASELINE config 5's law (power-law successor counts k^-1.5 on [1, 4096], 4 actions, discounted reward
    gamma = 0.95, eps = 1e-6, Pessimistic + Maximize synthesis) at `states` states, float64 and float32:
    the counter generator's columns (oracle.Model.generate == engine.generate_host) solved by the reference's
    control_synthesis.  Whole vectors and policies are stored (c5s.npz)."""
    import time
    res = {"config": dict(states=states, actions=4, law=1, alpha=1.5, kmax=4096, seed=1, discount=0.95,
                          eps=1e-6, rewards="np.random.default_rng(1).random(states).astype(dtype)"),
           "runs": {}}
    full = {}
    for dt in (np.float64, np.float32):
        name = "f64" if dt == np.float64 else "f32"
        rm = Model.generate(states, 4, law=1, alpha=1.5, kmax=4096, seed=1, dtype=dt)
        r = np.random.default_rng(1).random(states).astype(dt)
        pr = Problem(oracle.INFINITE_REWARD, rewards=r, discount=0.95, eps=1e-6, pessimistic=True, maximize=True)
        t = time.time()
        out = rm.solve(pr, synthesize=True)
        res["runs"][name] = {"iterations": int(out["iterations"]), "seconds": time.time() - t,
                             "threads": os.cpu_count(), "nnz": int(rm.sizes()[2]),
                             "values_sha256": digest(out["values"]), "residual_sha256": digest(out["residual"]),
                             "policy_sha256": digest(out["policy"].astype(np.int32))}
        full[f"{name}/values"] = out["values"]
        full[f"{name}/residual"] = out["residual"]
        full[f"{name}/policy"] = out["policy"].astype(np.int32)
        print("c5s", name, out["iterations"], flush=True)
    with open(os.path.join(OUT, "c5s.json"), "w") as f:
        json.dump(res, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "c5s.npz"), **full)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true")
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--c5s", action="store_true")
    ap.add_argument("--no-small", action="store_true")
    a = ap.parse_args()
    oracle.build()
    if not a.no_small:
        small()
    if a.c2:
        big("c2")
    if a.c3:
        big("c3")
    if a.c5s:
        c5_scaled()
