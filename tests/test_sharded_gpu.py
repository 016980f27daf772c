"""The sharded path on the device: shard stores (rimdp_model_create_shard /
generated shards), padded value buffers and the external stop test (global
residual from the gathered iterates), driven (a) by ShardedSolver over a 1-rank NCCL group and (b) as
two shards in lockstep on one GPU with the exchange done by device copies —
both bit-identical to the unsharded solve."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2401_04068_b200 import engine, problems as P, sharded

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a).view(np.uint64)


@pytest.fixture(scope="module")
def model_arrays():
    return engine.random_imdp(1001, 3, 24.0 / 1001, 1.0 / 24, 7)


def plans(n):
    goal = np.zeros(n, np.uint8)
    goal[-10:] = 1
    rew = np.random.default_rng(2).random(n)
    return [dict(initial=goal.astype(np.float64), frozen=goal, finite=False, eps=1e-6, pessimistic=True,
                 maximize=True),
            dict(initial=goal.astype(np.float64), frozen=goal, finite=True, horizon=17, pessimistic=False,
                 maximize=False),
            dict(initial=rew, rewards=rew, discount=0.95, finite=False, eps=1e-6, pessimistic=True, maximize=False)]


def test_one_rank_nccl_group_matches_engine_solve(model_arrays):
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = len(model_arrays[0]) - 1
        for plan in plans(n):
            ref = engine.DeviceModel.from_csc(*model_arrays).solve(**plan)
            shard = sharded.DeviceShard(engine.DeviceModel.from_csc(*model_arrays), 0, 1, n)
            out = sharded.ShardedSolver(shard, chunk=7).solve(**plan)
            assert out.iterations == ref["iterations"]
            assert np.array_equal(bits(out.values), bits(ref["values"]))
            assert np.array_equal(bits(out.residual), bits(ref["residual"]))
    finally:
        dist.destroy_process_group()


def lockstep(shards, plan, chunk=5):
    """Two shards of one GPU advanced in lockstep, exchanging slices with device copies."""
    for sh in shards:
        sh.begin(**plan)
    total = plan["horizon"] if plan["finite"] else 1_000_000
    k, done = 0, False
    while k < total and not done:
        for _ in range(chunk):
            k += 1
            for sh in shards:
                sh.advance()
            torch.cuda.synchronize()
            S = shards[0].S
            for dst in shards:
                for src in shards:
                    if src is not dst:
                        dst.values[k & 1][src.rank * S:(src.rank + 1) * S].copy_(
                            src.values[k & 1][src.rank * S:(src.rank + 1) * S])
            torch.cuda.synchronize()
            # no residual exchange: the stop test reduces the gathered iterates itself
            for sh in shards:
                sh.stop_test()
        states = [sh.poll() for sh in shards]
        assert len({(a, b) for a, b, _ in states}) == 1
        done = states[0][1]
    return [sh.finish() for sh in shards]


@pytest.mark.parametrize("source", ["csc", "generated"])
def test_two_shards_in_lockstep_bit_identical(model_arrays, source):
    if source == "csc":
        arrays = model_arrays
        n = len(arrays[0]) - 1
        whole = engine.DeviceModel.from_csc(*arrays)
        parts = [engine.DeviceModel.from_csc_shard(*sharded.slice_csc(*arrays, sb, se), sb, n)
                 for sb, se in sharded.shard_ranges(n, 2)]
    else:
        n = 1501
        whole = engine.DeviceModel.generate(engine.gen_config(n, 4, law=1, kmax=700, seed=3))
        parts = [engine.DeviceModel.generate(engine.gen_config(n, 4, law=1, kmax=700, seed=3, state_begin=sb,
                                                               state_end=se))
                 for sb, se in sharded.shard_ranges(n, 2)]
    shards = [sharded.DeviceShard(m, r, 2, n) for r, m in enumerate(parts)]
    for plan in plans(n):
        ref = whole.solve(**plan)
        outs = lockstep(shards, plan)
        for o in outs:
            assert o["iterations"] == ref["iterations"]
            assert np.array_equal(bits(o["values"][:n]), bits(ref["values"]))
