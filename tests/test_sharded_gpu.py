"""The sharded path on the device, all bit-identical to the
unsharded solve (sharding changes no per-state arithmetic):

* two and three processes sharing GPU 0, each holding one state shard
  (rimdp_model_create_shard / generated shards, one rank owning no state),
  exchanging V through the fused peer stores of the action kernel over CUDA
  IPC windows, with the peer_sync_stop stop test — the multi-process driver
  of bench.py (sharded.PeerShard + ShardedSolver, gloo for the handle swap);
* the single-process multi-device C ABI (rimdp_multi_*, MultiModel) with
  two and three shards on device 0: value iteration, synthesis (stationary
  and time-dependent), policy verification, InfeasibleColumn and
  NonConvergence reports with global indices, float32;
* the unfused NCCL baseline (sharded.NcclShard) over a one-rank group."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2401_04068_b200 import engine, problems as P, sharded

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def csc_model():
    return engine.random_imdp(1001, 3, 24.0 / 1001, 1.0 / 24, 7)


def plans(n, dtype=np.float64):
    goal = np.zeros(n, np.uint8)
    goal[-10:] = 1
    rew = np.random.default_rng(2).random(n).astype(dtype)
    g = goal.astype(dtype)
    return [dict(initial=g, frozen=goal, finite=False, eps=1e-6, pessimistic=True, maximize=True),
            dict(initial=g, frozen=goal, finite=True, horizon=17, pessimistic=False, maximize=False),
            dict(initial=rew, rewards=rew, discount=0.95, finite=False, eps=1e-6, pessimistic=True, maximize=False)]


# ---- multi-process: one shard per process, CUDA IPC peer exchange ---------------------------------

def _rank_main(rank, world, port, source, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sb, se = sharded.shard_ranges(n, world)[rank]
        if source == "csc":
            m = engine.DeviceModel.from_csc_shard(*sharded.slice_csc(*csc_model(), sb, se), sb, n)
        else:
            m = engine.DeviceModel.generate(engine.gen_config(n, 4, law=1, kmax=700, seed=3, state_begin=sb,
                                                              state_end=se))
        solver = sharded.ShardedSolver(sharded.PeerShard(m, rank, world, n), chunk=9)
        outs = []
        for plan in plans(n):
            r = solver.solve(**plan)
            outs.append((r.values, r.residual, r.iterations))
        q.put((rank, outs))
        dist.barrier()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("source,world,n", [("csc", 2, 1001), ("generated", 3, 1501), ("csc", 4, 1001)])
def test_peer_exchange_processes_sharing_one_gpu(source, world, n):
    import torch.multiprocessing as mp
    if source == "csc":
        whole = engine.DeviceModel.from_csc(*csc_model())
    else:
        whole = engine.DeviceModel.generate(engine.gen_config(n, 4, law=1, kmax=700, seed=3))
    refs = [whole.solve(**plan) for plan in plans(n)]
    whole.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, source, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(got[r], str), got[r]
        for (v, res, it), ref in zip(got[r], refs):
            assert it == ref["iterations"]
            assert np.array_equal(bits(v), bits(ref["values"]))
            assert np.array_equal(bits(res), bits(ref["residual"]))
    assert all(p.exitcode == 0 for p in procs)


# ---- single process, several shards: rimdp_multi_* ----------------------------------------------

@pytest.mark.parametrize("world", [2, 3])
def test_multi_model_solves_bit_identical(world):
    arrays = csc_model()
    n = len(arrays[0]) - 1
    whole = engine.DeviceModel.from_csc(*arrays)
    mm = engine.MultiModel(*arrays, world=world, devices=[0] * world)
    cut = mm.info()["state_begin"]
    assert cut[0] == 0 and cut[-1] == n and np.all(np.diff(cut) >= 0)
    for plan in plans(n):
        for record in ("none", "last") + (("all",) if plan["finite"] else ()):
            a, b = whole.solve(record=record, **plan), mm.solve(record=record, **plan)
            assert a["iterations"] == b["iterations"]
            assert np.array_equal(bits(a["values"]), bits(b["values"]))
            assert np.array_equal(bits(a["residual"]), bits(b["residual"]))
            if record != "none":
                assert np.array_equal(a["chosen"], b["chosen"])
    # through the reference-mirroring API: synthesis, then verification of the policy (forced columns)
    spec = P.Specification(P.InfiniteTimeReachability(list(range(n - 10, n)), 1e-6))
    pol_a, vf_a = P.control_synthesis(whole, spec, arrays[0])
    pol_b, vf_b = P.control_synthesis(mm, spec, arrays[0])
    assert np.array_equal(pol_a.columns, pol_b.columns) and np.array_equal(bits(vf_a.values), bits(vf_b.values))
    va, vb = P.verify_policy(whole, pol_a, spec, arrays[0]), P.verify_policy(mm, pol_a, spec, arrays[0])
    assert va.iterations == vb.iterations and np.array_equal(bits(va.values), bits(vb.values))
    mm.close()
    whole.close()


def test_multi_model_errors_carry_global_indices():
    sp, cp, rv, lo, up = csc_model()
    n = len(sp) - 1
    up = up.copy()
    bad = int(sp[800]) + 1                 # a column of a late state: in the last shard
    up[cp[bad]:cp[bad + 1]] = lo[cp[bad]:cp[bad + 1]]  # upper bounds sum below 1
    whole = engine.DeviceModel.from_csc(sp, cp, rv, lo, up)
    mm = engine.MultiModel(sp, cp, rv, lo, up, world=3, devices=[0, 0, 0])
    goal = np.zeros(n, np.uint8)
    goal[-10:] = 1
    kw = dict(initial=goal.astype(np.float64), frozen=goal, finite=False, eps=1e-6)
    errs = []
    for m in (whole, mm):
        with pytest.raises(engine.EngineError) as e:
            m.solve(**kw)
        errs.append((e.value.status, e.value.column, e.value.message))
    assert errs[0] == errs[1] and errs[0][1] == bad
    ok = engine.MultiModel(*csc_model(), world=2, devices=[0, 0])
    for m in (engine.DeviceModel.from_csc(*csc_model()), ok):
        with pytest.raises(engine.EngineError) as e:
            m.solve(initial=goal.astype(np.float64), frozen=goal, finite=False, eps=1e-300, max_iterations=5)
        assert e.value.status == engine.ERR_NON_CONVERGENCE and e.value.iterations == 5


def test_multi_model_float32_power_law():
    arrays = engine.generate_host(engine.gen_config(3000, 4, law=1, kmax=2048, seed=5, dtype=np.float32))
    n = 3000
    whole = engine.DeviceModel.from_csc(*arrays)
    mm = engine.MultiModel(*arrays, world=2, devices=[0, 0])
    for plan in plans(n, np.float32):
        a, b = whole.solve(record="last", **plan), mm.solve(record="last", **plan)
        assert a["iterations"] == b["iterations"]
        assert np.array_equal(bits(a["values"]), bits(b["values"])) and np.array_equal(a["chosen"], b["chosen"])


# ---- the unfused baseline --------------------------------------------------------------------------

def test_one_rank_nccl_baseline_matches_engine_solve():
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        arrays = csc_model()
        n = len(arrays[0]) - 1
        for plan in plans(n):
            ref = engine.DeviceModel.from_csc(*arrays).solve(**plan)
            shard = sharded.NcclShard(engine.DeviceModel.from_csc(*arrays), 0, 1, n)
            out = sharded.ShardedSolver(shard, chunk=7).solve(**plan)
            assert out.iterations == ref["iterations"]
            assert np.array_equal(bits(out.values), bits(ref["values"]))
            assert np.array_equal(bits(out.residual), bits(ref["residual"]))
    finally:
        dist.destroy_process_group()


def test_connected_shard_refuses_lone_solves():
    """A shard connected to peers iterates only together with them: a lone rimdp_solve / bellman_step is
    refused (it would wait forever for the peers' flags); column values need no exchange and still work."""
    arrays = csc_model()
    n = len(arrays[0]) - 1
    parts = [engine.DeviceModel.from_csc_shard(*sharded.slice_csc(*arrays, sb, se), sb, n)
             for sb, se in sharded.shard_ranges(n, 2)]
    for p in parts:
        p.set_value_capacity(n)
    engine.connect_local(parts)
    goal = np.zeros(n, np.uint8)
    goal[-10:] = 1
    for call in (lambda: parts[0].solve(initial=goal.astype(np.float64), frozen=goal, finite=True, horizon=3),
                 lambda: parts[1].bellman_step(goal.astype(np.float64))):
        with pytest.raises(engine.EngineError) as e:
            call()
        assert e.value.status == engine.ERR_INVALID_ARGUMENT and "connected shard" in e.value.message
    q = parts[0].column_values(np.random.default_rng(1).random(n))
    ref = engine.DeviceModel.from_csc(*arrays).column_values(np.random.default_rng(1).random(n))
    assert np.array_equal(bits(q), bits(ref[:len(q)]))
