#!/usr/bin/env python
"""Benchmark: transitions/s per robust Bellman iteration on BASELINE config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference] [--config c2|c3|...]

A "step" is one robust Bellman iteration (column O-max kernels + fused
action/residual kernel) over the whole transition store.  `value` is
whole-job transitions/s with the model resident in HBM (CUDA events on the
model stream, max over ranks); `e2e` is the same metric through the public
solve call with host buffers (model upload, plan upload, full solve to
convergence, result download), the headline against the reference arm.
`cpu_baseline` times the reference itself (oracle/_ref, all host threads) on
a bounded sample of the same workload.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # SURVEY §8(d) synthetic inputs; the generator is the reference's own law
    "c2": dict(desc="C2: random_imdp 100000 states x 4 actions x 32 successors (12.8M transitions), "
                    "Pmaxmin InfiniteTimeReachability(goal = last 1% of states, eps = 1e-6), f64",
               states=100000, actions=4, density=32.0 / 100000, scale=1.0 / 32, seed=1, goal_frac=0.01,
               pessimistic=True, maximize=True, eps=1e-6),
    "c3": dict(desc="C3: random_imdp 2000 states x 10 actions x 2000 successors (40M transitions), "
                    "Pminmin InfiniteTimeReachability(goal = last 1%, eps = 1e-6), f64",
               states=2000, actions=10, density=1.0, scale=1.0 / 2000, seed=1, goal_frac=0.01,
               pessimistic=True, maximize=False, eps=1e-6),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons, sampled every 20 ms from before the
    timed region until after the last GPU phase (timed region, kernel-timing
    pass and the end-to-end solve): every sample after the "timed" mark is
    taken under load."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.lines = []
        self.marks = {}

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, name):
        self.marks[name] = time.perf_counter()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.proc = None

    def summary(self):
        t0 = self.marks.get("timed", 0.0)
        t1 = self.marks.get("end", float("inf"))
        sm, mx, reasons, inside = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6 or ts < t0:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            inside += ts <= t1 + 0.02
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_in_timed_region": inside,
                "window": "timed region through kernel-timing pass and end-to-end solve (GPU busy)"}


def make_problem(w):
    n = w["states"]
    goal = list(range(n - int(round(n * w["goal_frac"])), n))
    return goal


def engine_arm(args, w):
    import torch
    from paper_2401_04068_b200 import engine, problems as P

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t0 = time.time()
    arrays = engine.random_imdp(w["states"], w["actions"], w["density"], w["scale"], w["seed"])
    sp, cp, rv, lo, up = arrays
    nnz = int(cp[-1])
    log(f"[bench] generated {w['states']} states, {nnz} transitions in {time.time() - t0:.1f}s")
    goal = make_problem(w)
    n = w["states"]
    spec = P.Specification(P.InfiniteTimeReachability(goal, w["eps"]),
                           P.PESSIMISTIC if w["pessimistic"] else P.OPTIMISTIC,
                           P.MAXIMIZE if w["maximize"] else P.MINIMIZE)
    plan = P.make_plan(spec, n, np.float64)

    # ---- resident throughput (value) ------------------------------------
    m = engine.DeviceModel.from_csc(sp, cp, rv, lo, up, device=local)
    stream = torch.cuda.ExternalStream(m.stream(), device=torch.device("cuda", local))
    total = args.warmup + args.steps
    kw = dict(initial=plan.initial, frozen=plan.frozen, finite=True, horizon=total + 1,
              pessimistic=w["pessimistic"], maximize=w["maximize"])
    clk = ClockSampler(local).__enter__()  # sampled through every GPU phase below
    time.sleep(0.3)  # let nvidia-smi start sampling before the GPU work begins
    m.begin(**kw)
    m.advance(args.warmup)
    m.poll()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk.mark("timed")
    start.record(stream)
    m.advance(args.steps)
    end.record(stream)
    torch.cuda.synchronize()
    clk.mark("end")
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    k_done, _, _ = m.poll()
    assert k_done == total, (k_done, total)
    ms_per_step = ms / args.steps

    # ---- dominant kernel timing (separate pass, events per launch) ------
    m.begin(**kw)
    m.advance(args.warmup)
    m.poll()
    m.profile(True)
    m.profile_read()
    prof_iters = min(args.steps, 200)
    m.advance(prof_iters)
    fused_ms, cols_ms, act_ms, it, kpi = m.profile_read()
    m.profile(False)
    m.finish()
    fused_avg, cols_avg, act_avg = fused_ms / it, cols_ms / it, act_ms / it
    if fused_avg >= cols_avg:
        kernel_name, kernel_avg = "bellman_short (fused column O-max + action + residual)", fused_avg
    else:
        kernel_name, kernel_avg = "omax_long/omax_short (per-column O-max of long states)", cols_avg
    es = 8
    alg_bytes = nnz * (4 + es + es + es)  # index + lower + gap + V gather
    peak, peak_src = load_peaks()
    achieved = alg_bytes / (kernel_avg * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get(args.config, {}).get("dram_bytes_per_launch")
    info = m.info()
    m.close()

    # ---- end to end through the public API with host buffers ------------
    torch.cuda.synchronize()
    t = time.perf_counter()
    dm = engine.DeviceModel.from_csc(sp, cp, rv, lo, up, device=local)
    vf = P.value_iteration(dm, spec)
    e2e_s = time.perf_counter() - t
    dm.close()
    h2d = sp.nbytes + cp.nbytes + rv.nbytes + lo.nbytes + up.nbytes + plan.initial.nbytes + plan.frozen.nbytes
    d2h = vf.values.nbytes + vf.residual.nbytes
    e2e_iters = vf.iterations
    ref_iters = None
    bit_exact = None
    gj = os.path.join(ROOT, "tests", "golden", f"{args.config}.json")
    if os.path.exists(gj):
        import hashlib
        with open(gj) as f:
            run = json.load(f)["runs"].get(f"m{int(w['maximize'])}p{int(w['pessimistic'])}")
        if run:
            ref_iters = run["iterations"]
            bit_exact = (hashlib.sha256(vf.values.tobytes()).hexdigest() == run["values_sha256"] and
                         hashlib.sha256(vf.residual.tobytes()).hexdigest() == run["residual_sha256"])

    clk.__exit__()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(arrays, w, plan, budget_s=args.cpu_budget)

    clocks = clk.summary()
    out = {
        "metric": "transitions/sec per Bellman iteration",
        "value": nnz * world / (ms_per_step * 1e-3),
        "unit": "transitions/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference random_imdp law, seed 1; generated on host, resident in HBM)",
        "config": {"workload": w["desc"], "states": n, "columns": int(len(cp) - 1), "transitions": nnz,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "per-iteration inputs (28 B x transitions) exceed the 126 MB L2; no flush needed",
                   "scheduler": {"short_columns": info.short_columns, "long_columns": info.long_columns}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": kernel_name,
                     "algorithmic_bytes_per_launch": alg_bytes, "launch_ms": kernel_avg,
                     "phase_ms": {"fused_short_states": fused_avg, "column_kernels": cols_avg,
                                  "action_kernel": act_avg},
                     "kernel_share_of_step": kernel_avg / max(fused_avg + cols_avg + act_avg, 1e-12),
                     "peak_source": peak_src},
        "e2e": {"value": nnz * e2e_iters / e2e_s, "unit": "transitions/s", "h2d_bytes_per_step": h2d / e2e_iters,
                "d2h_bytes_per_step": d2h / e2e_iters, "seconds_to_convergence": e2e_s, "iterations": e2e_iters,
                "reference_iterations": ref_iters, "values_bit_exact_vs_reference": bit_exact, "call": "DeviceModel.from_csc + problems.value_iteration (C ABI)"},
        "time_to_convergence_s": e2e_s,
        "gpu_launches": args.steps * kpi,
        "clocks": clocks,
    }
    if cpu:
        out["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


_CPU_MODELS: dict = {}


def cpu_sample(arrays, w, plan, budget_s=15.0, which=None, model_cache=True):
    """The reference (oracle/_ref, all host threads) on a bounded number of
    iterations of the same workload; the oracle port (1 thread) if the
    reference library is absent."""
    import oracle
    sp, cp, rv, lo, up = arrays
    which = which or ("ref" if oracle.ref_available() else "port")
    if which == "port" and not oracle.port_available():
        oracle.build(ref=False)
    cores = os.cpu_count() if which == "ref" else 1
    key = (which, id(arrays))
    m = _CPU_MODELS.get(key) if model_cache else None
    if m is None:
        t = time.time()
        m = oracle.Model.from_arrays(which, sp, cp, rv, lo, up)
        log(f"[bench] cpu model ({which}) built in {time.time() - t:.1f}s")
        _CPU_MODELS[key] = m
    goal = np.nonzero(plan.frozen)[0].tolist()

    def run(k):
        pr = oracle.Problem(oracle.FINITE_REACH, reach=goal, horizon=k, pessimistic=w["pessimistic"],
                            maximize=w["maximize"])
        t0 = time.perf_counter()
        m.solve(pr, workers=0)
        return time.perf_counter() - t0

    one = run(1)
    k = max(1, min(200, int(budget_s / max(one, 1e-6))))
    secs = run(k)
    nnz = int(cp[-1])
    return {"value": nnz * k / secs, "unit": "transitions/s", "cores": cores,
            "kind": "reference" if which == "ref" else "port",
            "sample": f"{k} Bellman iterations of the same workload (FiniteTimeReachability horizon {k}, "
                      f"same goal set and modes), value_iteration with workers=0, {secs:.2f}s"}


def reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2401_04068_b200 import engine
    arrays = engine.random_imdp(w["states"], w["actions"], w["density"], w["scale"], w["seed"])
    from paper_2401_04068_b200 import problems as P
    goal = make_problem(w)
    spec = P.Specification(P.InfiniteTimeReachability(goal, w["eps"]))
    plan = P.make_plan(spec, w["states"], np.float64)
    target = min(3.0, 120.0 / max(1, args.steps))
    cpu = None
    for _ in range(args.warmup and 1):
        cpu = cpu_sample(arrays, w, plan, budget_s=target)
    vals = []
    for _ in range(args.steps):
        cpu = cpu_sample(arrays, w, plan, budget_s=target, model_cache=True)
        vals.append(cpu["value"])
    v = statistics.median(vals)
    nnz = int(arrays[1][-1])
    cpu["value"] = v
    out = {"impl": "reference", "metric": "transitions/sec per Bellman iteration", "value": v,
           "unit": "transitions/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": nnz / v * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference random_imdp law, seed 1)",
           "config": {"workload": w["desc"], "states": w["states"], "transitions": nnz,
                      "parallelism": "host threads"},
           "cpu_baseline": cpu,
           "e2e": {"value": v, "unit": "transitions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU reference work")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = WORKLOADS[args.config]
    if args.impl == "reference":
        reference_arm(args, w)
    else:
        engine_arm(args, w)


if __name__ == "__main__":
    main()
