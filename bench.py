#!/usr/bin/env python
"""Benchmark: transitions/s per robust Bellman iteration (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
                    [--config c2|c3|c4|c5] [--dtype f64|f32]

A "step" is one robust Bellman iteration over the whole transition store:
the column O-max kernels, the fused action/update/residual kernel and, at
N > 1, the value all-gather + residual all-reduce of the state-sharded
solve.  The default workload is BASELINE config 2 (configs[1], the one the
metric is quoted on that fits one GPU).

  value     whole-job transitions/s, model resident in HBM, CUDA events on the
            model stream around exactly K steps (max over ranks at N > 1)
  e2e       the same metric through the public solve call with host buffers:
            model upload (host-generated configs) + plan upload + solve to
            convergence + result download, divided over the iterations
  roofline  the column phase (the dominant kernels) against HBM: algorithmic
            bytes = transitions x (index + lower + gap + V gather) per launch
             / its event-timed duration
  cpu_baseline  the reference itself (oracle/_ref, all host threads) on a
            bounded sample of the same workload (rank 0, N = 1)

See DESIGN.md "Measurement".
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
    # SURVEY §8(d) synthetic inputs
    "c2": dict(desc="C2: random_imdp 100000 states x 4 actions x 32 successors (12.8M transitions), "
                    "Pmaxmin InfiniteTimeReachability(goal = last 1% of states, eps = 1e-6)",
               source="reference", states=100000, actions=4, density=32.0 / 100000, scale=1.0 / 32, seed=1,
               kind="reach", goal_frac=0.01, pessimistic=True, maximize=True, eps=1e-6,
               sample=None, weak_support=32),
    "c3": dict(desc="C3: random_imdp 2000 states x 10 actions x 2000 successors (40M transitions), "
                    "Pminmin InfiniteTimeReachability(goal = last 1%, eps = 1e-6), long-column path",
               source="reference", states=2000, actions=10, density=1.0, scale=1.0 / 2000, seed=1,
               kind="reach", goal_frac=0.01, pessimistic=True, maximize=False, eps=1e-6, sample=None),
    "c4": dict(desc="C4: 10M states x 8 actions x 64 successors (5.12e9 transitions, counter-based generator "
                    "in HBM), Pmaxmin InfiniteTimeReachability(goal = last 1%, eps = 1e-6)",
               source="generated", states=10_000_000, actions=8, law=0, support=64, seed=1,
               kind="reach", goal_frac=0.01, pessimistic=True, maximize=True, eps=1e-6,
               sample=dict(states=100_000)),
    "c5": dict(desc="C5: 1M states x 4 actions, power-law successor counts k^-1.5 on [1, 4096] (~2e8 "
                    "transitions, generated in HBM), discounted reward gamma = 0.95, Pmax strategy synthesis, "
                    "eps = 1e-6",
               source="generated", states=1_000_000, actions=4, law=1, alpha=1.5, kmax=4096, seed=1,
               kind="reward", discount=0.95, pessimistic=True, maximize=True, eps=1e-6,
               sample=dict(states=50_000), host_arrays=True),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def scaled_workload(w, world, scaling):
    """The workload at `world` GPUs.  Weak scaling (the default for C2, the
    default config): the same law with world x the states, so every GPU
    keeps C2's 100000 states x 4 actions x 32 successors.  At N > 1 the
    columns come from the counter generator with random_imdp's value law
    (lower = u/32, upper = min(lower + v (1 - 1/32), 1)), each rank
    generating only its own shard in HBM — random_imdp's sequential
    mt19937_64 stream would make every rank build the whole N x model on the
    host.  Configs 3-5 are fixed-size (C4 is already the 8-GPU shard config):
    strong scaling."""
    if scaling == "weak" and world > 1 and w.get("weak_support"):
        n = w["states"] * world
        k = w["weak_support"]
        w = dict(w, states=n, source="generated", law=0, support=k, sample=dict(states=w["states"]), host_arrays=True,
                 desc=w["desc"].split(":")[0] + f" law weak-scaled x{world}: {n} states x {w['actions']} actions x "
                      f"{k} successors (counter generator, random_imdp's value law; each rank generates only its "
                      "shard, on the host, and uploads it), Pmaxmin InfiniteTimeReachability(goal = last 1%, eps = 1e-6)")
        return w, "weak"
    return w, ("weak" if (w.get("weak_support") and scaling == "weak") else "strong")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "of measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "of fallback (B200_PROFILING.md 6.65 TB/s; MEASURED_PEAKS.json absent)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons every 20 ms from before the timed
    region until after the last GPU phase; samples after the "timed" mark are
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
            # nvidia-smi takes a few hundred ms to start: wait for its first sample (at most 3 s), so that a
            # short timed region (C2: ~20 ms) is covered by the 20 ms sampling
            t_end = time.perf_counter() + 3.0
            while not self.lines and time.perf_counter() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
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
                "window": "timed region through the kernel-timing pass (GPU busy); stopped before the "
                          "end-to-end solve"}


# ---------------------------------------------------------------------------
# workloads

def goal_states(n, frac):
    return np.arange(n - int(round(n * frac)), n)


def rewards_for(n, seed):
    return np.random.default_rng(seed).random(n)


def gen_cfg(w, dtype, states=None, device=0, state_begin=0, state_end=0):
    from paper_2401_04068_b200 import engine
    return engine.gen_config(states or w["states"], w["actions"], law=w["law"], support=w.get("support", 64),
                             alpha=w.get("alpha", 1.5), kmax=w.get("kmax", 4096), seed=w["seed"], dtype=dtype,
                             device=device, state_begin=state_begin, state_end=state_end)


def pin_arrays(arrays):
    """The e2e leg's host CSC arrays in page-locked memory (what a serving process keeps its models in; the
    contract's "pinned host memory"): the upload is then one DMA per array.  Pinning happens before the
    timed region; if the host refuses, the arrays stay pageable (staged upload) and the line says so."""
    import torch
    try:
        out = tuple(torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in arrays)
        return out, "pinned"
    except RuntimeError as e:
        log(f"[bench] pinning the host arrays failed ({e}); pageable upload")
        return arrays, "pageable"


def host_arrays(w, dtype, states=None):
    """Host CSC arrays of the workload (or of its down-scaled CPU sample)."""
    from paper_2401_04068_b200 import engine
    if w["source"] == "reference":
        return engine.random_imdp(states or w["states"], w["actions"], w["density"], w["scale"], w["seed"],
                                  dtype=dtype)
    return engine.generate_host(gen_cfg(w, dtype, states=states))


def plan_kw(w, n, dtype):
    """The marshalled plan (solver.hpp:40-80) of the workload's specification."""
    dt = np.dtype(dtype)
    if w["kind"] == "reach":
        frozen = np.zeros(n, np.uint8)
        frozen[goal_states(n, w["goal_frac"])] = 1
        return dict(initial=frozen.astype(dt), frozen=frozen, pessimistic=w["pessimistic"], maximize=w["maximize"],
                    eps=float(dt.type(w["eps"])))
    r = rewards_for(n, w["seed"]).astype(dt)
    return dict(initial=r, rewards=r, discount=float(dt.type(w["discount"])), pessimistic=w["pessimistic"],
                maximize=w["maximize"], eps=float(dt.type(w["eps"])))


def spec_for(w, n, dtype):
    from paper_2401_04068_b200 import problems as P
    sat = P.PESSIMISTIC if w["pessimistic"] else P.OPTIMISTIC
    strat = P.MAXIMIZE if w["maximize"] else P.MINIMIZE
    if w["kind"] == "reach":
        return P.Specification(P.InfiniteTimeReachability(list(goal_states(n, w["goal_frac"])), w["eps"]), sat, strat)
    return P.Specification(P.InfiniteTimeReward(rewards_for(n, w["seed"]).astype(dtype), w["discount"], w["eps"]),
                           sat, strat)


# ---------------------------------------------------------------------------
# engine arm

def build_model(w, dtype, rank, world, local):
    """This rank's store: the whole model (N = 1) or its state shard."""
    from paper_2401_04068_b200 import engine, sharded
    n = w["states"]
    sb, se = sharded.shard_ranges(n, world)[rank]
    t0 = time.time()
    arrays = None  # this rank's host CSC arrays (the whole model at N = 1, the shard at N > 1)
    if w["source"] == "reference":
        arrays = host_arrays(w, dtype)
        if world == 1:
            m = engine.DeviceModel.from_csc(*arrays, device=local)
        else:
            arrays = sharded.slice_csc(*arrays, sb, se)
            m = engine.DeviceModel.from_csc_shard(*arrays, sb, n, device=local)
    elif w.get("host_arrays"):
        # the counter generator on the host for this rank's states only, uploaded like a caller's arrays
        # (so the end-to-end number includes the host -> device copy of the store)
        arrays = engine.generate_host(gen_cfg(w, dtype, state_begin=sb if world > 1 else 0,
                                              state_end=se if world > 1 else 0))
        if world == 1:
            m = engine.DeviceModel.from_csc(*arrays, device=local)
        else:
            m = engine.DeviceModel.from_csc_shard(*arrays, sb, n, device=local)
    else:
        cfg = gen_cfg(w, dtype, device=local, state_begin=sb if world > 1 else 0, state_end=se if world > 1 else 0)
        m = engine.DeviceModel.generate(cfg)
    log(f"[bench] rank {rank}: states [{sb}, {se}), {m.nnz} transitions built in {time.time() - t0:.1f}s")
    return m, arrays


def engine_arm(args, w):
    import torch
    from paper_2401_04068_b200 import engine, problems as P, sharded

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RIMDP_BENCH_DEVICE_MAP=0,0 (tests on a one-GPU box): local rank r runs on device map[r]
    dmap = os.environ.get("RIMDP_BENCH_DEVICE_MAP")
    if dmap:
        local = int(dmap.split(",")[local])
    torch.cuda.set_device(local)
    dist = None
    if world > 1 and args.exchange == "peer":
        # the fused exchange stores into the peers' HBM: every pair of the node's GPUs needs P2P access
        # (NVLink / NVSwitch).  Without it every rank takes the NCCL path (the same check on every rank)
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        devs = [int(dmap.split(",")[r]) for r in range(local_world)] if dmap else list(range(local_world))
        if any(a != b and not torch.cuda.can_device_access_peer(a, b) for a in devs for b in devs):
            log("[bench] no P2P access between the node's GPUs: NCCL exchange instead of the fused peer stores")
            args.exchange = "nccl"
    if world > 1:
        import torch.distributed as dist
        # control plane only (IPC handle swap, barriers, max over ranks): gloo on host tensors.  The peer
        # exchange needs no collective library; the NCCL baseline needs NCCL for its all-gather.
        if args.exchange == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dtype = np.float64 if args.dtype == "f64" else np.float32
    es = np.dtype(dtype).itemsize
    n = w["states"]
    m, arrays = build_model(w, dtype, rank, world, local)
    host_kind = "pageable"
    if arrays is not None and not args.no_e2e:
        arrays, host_kind = pin_arrays(arrays)
    local_nnz = m.nnz
    total_nnz = local_nnz
    if world > 1:
        t = torch.tensor([local_nnz, local_nnz], dtype=torch.int64, device="cuda" if args.exchange == "nccl" else "cpu")
        dist.all_reduce(t[:1], op=dist.ReduceOp.SUM)
        dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
        total_nnz, max_nnz = int(t[0]), int(t[1])
    kw = plan_kw(w, n, dtype)
    total = args.warmup + args.steps
    run_kw = dict(kw, finite=True, horizon=total + 1)  # a fixed number of iterations: no early stop
    stream = torch.cuda.ExternalStream(m.stream(), device=torch.device("cuda", local))
    clk = ClockSampler(local).__enter__()
    time.sleep(0.3)

    # ---- resident throughput (value) ------------------------------------
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world == 1:
        m.begin(**run_kw)
        m.advance(args.warmup)
        m.poll()
        torch.cuda.synchronize()
        clk.mark("timed")
        start.record(stream)
        m.advance(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        k_done, _, _ = m.poll()
        assert k_done == total, (k_done, total)
    else:
        # the state-sharded solve: V exchanged by the action kernel's peer stores (sharded.PeerShard), or
        # the unfused NCCL all-gather baseline with --exchange nccl
        shard = (sharded.PeerShard if args.exchange == "peer" else sharded.NcclShard)(m, rank, world, n)
        shard.begin(**run_kw)
        shard.advance(args.warmup)
        shard.poll()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        clk.mark("timed")
        start.record(stream)
        shard.advance(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        k_done, _, _ = shard.poll()
        assert k_done == total, (k_done, total)
        m.finish()
    clk.mark("end")
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device="cuda" if args.exchange == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps

    # ---- dominant kernels: the column phase, event-timed per launch ------
    if world > 1:
        shard.begin(**run_kw)  # includes the barrier after the windows are reset
    else:
        m.begin(**run_kw)
    m.advance(args.warmup)
    m.poll()
    m.profile(True)
    m.profile_read()
    prof_iters = min(args.steps, 200)
    if world > 1 and args.exchange == "nccl":
        shard.advance(prof_iters)
    else:
        m.advance(prof_iters)
    fused_ms, cols_ms, act_ms, it, kpi = m.profile_read()
    m.profile(False)
    m.finish()
    fused_avg, cols_avg, act_avg = fused_ms / it, cols_ms / it, act_ms / it
    info = m.info()
    if fused_avg >= cols_avg:
        kernel_name, kernel_avg = "bellman_short (fused column O-max + action + residual)", fused_avg
    else:
        kernel_name, kernel_avg = "column O-max phase (omax_short / omax_long / omax_sorted launches)", cols_avg
    alg_bytes = local_nnz * (4 + es + es + es)  # index + lower + gap + V gather
    peak, peak_src = load_peaks()
    achieved = alg_bytes / (kernel_avg * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get(f"{args.config}_{args.dtype}", {}).get("dram_bytes_per_launch")

    # ---- end to end through the public API with host buffers ------------
    # the clock sampler stops first: nvidia-smi's NVML queries contend with
    # the driver calls of the upload (measured: occasional 50 ms stalls)
    clk.__exit__()
    if arrays is not None and not args.no_e2e:
        # the resident benchmark model is released before the clock starts: the end-to-end model's allocation
        # then reuses its device memory instead of paying the first-touch mapping of fresh pages (measured:
        # 134 ms on the first process of a fresh box)
        m.close()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    h2d = sum(np.asarray(v).nbytes for v in kw.values() if isinstance(v, np.ndarray))
    if args.no_e2e:  # kernel experiments only: no solve to convergence
        e2e_iters, values, residual = 1, np.zeros(n, dtype), np.zeros(n, dtype)
    elif world == 1:
        if arrays is not None:
            dm = engine.DeviceModel.from_csc(*arrays, device=local)
            h2d += sum(a.nbytes for a in arrays)
        else:
            dm = m
        t_up = time.perf_counter()
        vf = P.value_iteration(dm, spec_for(w, n, dtype))
        e2e_iters, values, residual = vf.iterations, vf.values, vf.residual
        log(f"[bench] e2e: model upload {1e3 * (t_up - t):.1f} ms, solve {1e3 * (time.perf_counter() - t_up):.1f} ms")
    else:
        if arrays is not None:
            dm = engine.DeviceModel.from_csc_shard(*arrays, sharded.shard_ranges(n, world)[rank][0], n, device=local)
            h2d += sum(a.nbytes for a in arrays)
        else:
            dm = m
        sh = (sharded.PeerShard if args.exchange == "peer" else sharded.NcclShard)(dm, rank, world, n) \
            if dm is not m else shard
        res = sharded.ShardedSolver(sh).solve(finite=False, **kw)
        e2e_iters, values, residual = res.iterations, res.values, res.residual
    e2e_s = time.perf_counter() - t
    if world > 1:
        tt = torch.tensor([e2e_s], device="cuda" if args.exchange == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    d2h = values.nbytes + residual.nbytes
    ref_iters = bit_exact = sample_diff = None
    gj = os.path.join(ROOT, "tests", "golden", f"{args.config}.json")
    if os.path.exists(gj) and not args.no_e2e and args.dtype == "f64" and w["states"] == WORKLOADS[args.config]["states"]:
        import hashlib
        with open(gj) as f:
            run = json.load(f)["runs"].get(f"m{int(w['maximize'])}p{int(w['pessimistic'])}")
        if run:
            ref_iters = run["iterations"]
            bit_exact = (hashlib.sha256(values.tobytes()).hexdigest() == run["values_sha256"] and
                         hashlib.sha256(residual.tobytes()).hexdigest() == run["residual_sha256"])
            idx = np.array(run["sample_idx"])
            sample_diff = float(np.abs(values[idx] - np.array([float.fromhex(h) for h in run["sample_hex"]])).max())
    m.close()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(w, dtype, budget_s=args.cpu_budget)

    out = {
        "metric": "transitions/sec per Bellman iteration",
        "value": total_nnz / (ms_per_step * 1e-3),
        "unit": "transitions/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": args.scaling_kind,
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": data_desc(w) + ("; generated on host and uploaded, resident in HBM"
                                if w["source"] == "reference" or w.get("host_arrays") else
                                "; generated directly in HBM (the e2e number excludes the store's upload)"),
        "config": config_for(w, total_nnz, es, (f"state-sharded x{world}, V exchanged by "
                                                + ("fused peer stores (CUDA IPC, NVLink)" if args.exchange == "peer"
                                                   else "NCCL all-gather")) if world > 1 else "single GPU"),
        "scheduler": {"short_columns": info.short_columns, "exact_long_columns": info.mid_columns,
                      "sorted_long_columns": info.long_columns, "max_column_length": info.max_column_length},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": kernel_name,
                     "algorithmic_bytes_per_launch": alg_bytes, "launch_ms": kernel_avg,
                     "phase_ms": {"fused_short_states": fused_avg, "column_kernels": cols_avg,
                                  "action_kernel": act_avg},
                     "kernel_share_of_step": kernel_avg / max(fused_avg + cols_avg + act_avg, 1e-12),
                     "peak_source": peak_src,
                     # the same phase against its measured DRAM bytes (ncu, cold cache): below the algorithmic
                     # fraction when V gathers hit L2 (C2, C3: V in L2 / shared memory), above when they miss (C4)
                     "dram_achieved": (traffic / (kernel_avg * 1e-3) / 1e9) if traffic else None,
                     "dram_frac": (traffic / (kernel_avg * 1e-3) / 1e9 / peak) if traffic else None},
        "e2e": {"value": total_nnz * e2e_iters / e2e_s, "unit": "transitions/s",
                "h2d_bytes_per_step": h2d / max(e2e_iters, 1), "d2h_bytes_per_step": d2h / max(e2e_iters, 1),
                "seconds_to_convergence": e2e_s, "iterations": e2e_iters,
                "host_buffers": host_kind if arrays is not None else "model generated in HBM (not uploaded)",
                "reference_iterations": ref_iters, "values_bit_exact_vs_reference": bit_exact,
                "max_abs_diff_vs_reference_samples": sample_diff,
                "call": ("DeviceModel.from_csc + problems.value_iteration (C ABI)" if world == 1 else
                         "DeviceModel.from_csc_shard + sharded.ShardedSolver.solve (C ABI; V exchanged "
                         + ("by the action kernel's peer stores over CUDA IPC)" if args.exchange == "peer" else
                            "by NCCL all-gather)"))},
        "time_to_convergence_s": e2e_s,
        "gpu_launches": args.steps * kpi,  # kernels_per_iteration counts peer_sync_stop when sharded
        "clocks": clk.summary(),
    }
    if world > 1:
        out["shard_nnz_max_over_mean"] = max_nnz / (total_nnz / world)
    if cpu:
        out["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU reference (the checker, timed)

_CPU_MODELS: dict = {}


def cpu_model(w, dtype, states=None):
    """The workload as a reference model built by the reference itself (oracle/_ref): random_imdp
    (random_model.hpp:42-101) for configs 2-3, the counter generator's columns through the reference's
    checked constructors for configs 4-5.  Returns (model, transitions, states)."""
    import oracle
    n = states or w["states"]
    key = (w["desc"], n, np.dtype(dtype).str)
    if key not in _CPU_MODELS:
        t = time.time()
        if w["source"] == "reference":
            m = oracle.Model.random(n, w["actions"], w["density"] if n == w["states"] else w["density"] * w["states"] / n,
                                    w["scale"], w["seed"], dtype=dtype)
        else:
            m = oracle.Model.generate(n, w["actions"], law=w["law"], support=w.get("support", 64),
                                      alpha=w.get("alpha", 1.5), kmax=w.get("kmax", 4096), seed=w["seed"], dtype=dtype)
        _CPU_MODELS[key] = (m, m.sizes()[2], n)
        log(f"[bench] reference model ({n} states) built in {time.time() - t:.1f}s")
    return _CPU_MODELS[key]


def cpu_sample(w, dtype, budget_s=15.0):
    """The reference (oracle/_ref: the unmodified reference headers, value_iteration with workers = 0 = all
    host threads) on a bounded number of iterations of the workload (configs 4-5: of its law at the
    `sample` state count)."""
    import oracle
    if not oracle.ref_available():
        oracle.build(port=False)
    states = (w.get("sample") or {}).get("states")
    m, nnz, n = cpu_model(w, dtype, states)
    kw = plan_kw(w, n, dtype)

    def run(k):
        if w["kind"] == "reach":
            pr = oracle.Problem(oracle.FINITE_REACH, reach=list(np.nonzero(kw["frozen"])[0]), horizon=k,
                                pessimistic=w["pessimistic"], maximize=w["maximize"])
        else:
            pr = oracle.Problem(oracle.FINITE_REWARD, rewards=kw["rewards"], discount=kw["discount"], horizon=k,
                                pessimistic=w["pessimistic"], maximize=w["maximize"])
        t0 = time.perf_counter()
        m.solve(pr, workers=0)
        return time.perf_counter() - t0

    one = run(1)
    k = max(1, min(200, int(budget_s / max(one, 1e-6))))
    secs = run(k)
    scope = "the same workload" if not states else f"the same law at {n} states ({nnz} transitions)"
    return {"value": nnz * k / secs, "unit": "transitions/s", "cores": os.cpu_count(), "kind": "reference",
            "sample": f"{k} Bellman iterations of {scope} (finite-horizon {k}, same goal/reward and modes), "
                      f"reference value_iteration with workers=0 on {os.cpu_count()} host threads, {secs:.2f}s"}


def reference_arm(args, w):
    """The reference's own CPU implementation (oracle/_ref) on this arm's config; rank 0 only at N > 1.
    Imports nothing from the engine package."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    dtype = np.float64 if args.dtype == "f64" else np.float32
    es = np.dtype(dtype).itemsize
    target = min(3.0, 120.0 / max(1, args.steps))
    cpu = None
    for _ in range(args.warmup and 1):
        cpu = cpu_sample(w, dtype, budget_s=target)
    vals = []
    for _ in range(args.steps):
        cpu = cpu_sample(w, dtype, budget_s=target)
        vals.append(cpu["value"])
    v = statistics.median(vals)
    nnz_full = cpu_model(w, dtype)[1] if w["source"] == "reference" else full_transitions(w)
    cpu["value"] = v
    out = {"impl": "reference", "metric": "transitions/sec per Bellman iteration", "value": v,
           "unit": "transitions/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": nnz_full / v * 1e3,
           "higher_is_better": True, "scaling": args.scaling_kind, "vs_baseline": None, "dtype": args.dtype,
           "data": data_desc(w),
           "config": config_for(w, nnz_full, es, f"reference CPU, {os.cpu_count()} host threads"),
           "cpu_baseline": cpu,
           "e2e": {"value": v, "unit": "transitions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def full_transitions(w):
    """Transitions of a counter-generated workload at full size (configs 4-5): the generator's column
    lengths, summed on the host without building the columns."""
    import oracle
    return oracle.generate_nnz(w["states"], w["actions"], law=w["law"], support=w.get("support", 64),
                               alpha=w.get("alpha", 1.5), kmax=w.get("kmax", 4096), seed=w["seed"])


def data_desc(w):
    return ("synthetic (reference random_imdp law, seed 1)" if w["source"] == "reference" else
            "synthetic (counter-based generator, seed 1)")


def config_for(w, transitions, es, parallelism):
    """The `config` object of both arms (identical keys; only `parallelism` differs)."""
    return {"workload": w["desc"], "states": w["states"], "columns": w["states"] * w["actions"],
            "transitions": transitions, "parallelism": parallelism,
            "l2": ("per-iteration inputs (index + bounds, 20 B x transitions) exceed the 126 MB L2; no flush needed"
                   if transitions and transitions * (4 + 2 * es) > 126e6 else "inputs fit in L2 (reported as is)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU reference work")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="experiments: skip the end-to-end solve (no e2e number)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: V exchange of the sharded solve (fused peer stores, or the NCCL baseline)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak (C2 law, N x the states) or strong (fixed model)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver's own launch sets WORLD_SIZE)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        log("[bench] spawning", args.gpus, "ranks:", " ".join(cmd))
        sys.exit(subprocess.call(cmd))
    if args.warmup < 3:
        args.warmup = 3
    w, args.scaling_kind = scaled_workload(WORKLOADS[args.config], int(os.environ.get("WORLD_SIZE", "1")),
                                           args.scaling)
    if args.impl == "reference":
        reference_arm(args, w)
    else:
        engine_arm(args, w)


if __name__ == "__main__":
    main()
