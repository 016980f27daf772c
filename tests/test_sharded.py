"""Multi-process sharded driver (paper_2401_04068_b200/sharded.py) on CPU:
world_size 2 over gloo, with a test double for the device shard that computes
its states' rows with the CPU checker (oracle port).  Covers the partitioning,
the padded in-place all-gather of V, the external stop test on the
residual of the gathered iterates and NonConvergence — and that the sharded result is
bit-identical to the unsharded one (per-state arithmetic is unchanged)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2401_04068_b200 import engine, sharded


def test_shard_ranges_cover_states_in_equal_slices():
    for n, w in ((10, 3), (7, 8), (100000, 8), (1, 2), (16, 4)):
        rs = sharded.shard_ranges(n, w)
        assert len(rs) == w and rs[0][0] == 0 and rs[-1][1] == n
        S = sharded.slice_length(n, w)
        for r, (sb, se) in enumerate(rs):
            assert sb == min(n, r * S) and se - sb <= S
            if r:
                assert sb == rs[r - 1][1]


def test_slice_csc_rebases_pointers():
    sp, cp, rv, lo, up = engine.random_imdp(30, 3, 0.2, 0.2, 4)
    lsp, lcp, lrv, llo, lup = sharded.slice_csc(sp, cp, rv, lo, up, 10, 20)
    assert lsp[0] == 0 and len(lsp) == 11 and lcp[0] == 0 and lcp[-1] == len(lrv)
    b, e = cp[sp[10]], cp[sp[20]]
    assert np.array_equal(lrv, rv[b:e]) and np.array_equal(llo, lo[b:e])


def test_shard_balance_of_synthetic_laws():
    for law in (0, 1):
        cp = engine.generate_host(engine.gen_config(40000, 4, law=law, support=32, kmax=1024, seed=3))[1]
        state_nnz = np.diff(cp).reshape(-1, 4).sum(1)
        assert sharded.shard_balance(state_nnz, 8) < (1.001 if law == 0 else 1.1)


class CpuShard:
    """Test double of sharded.PeerShard: the same protocol (begin + barrier, advance(n), poll, finish) on
    the CPU.  The rows of states [sb, se) come from the oracle port's Bellman step; the exchange the engine
    fuses into its action kernel (peer stores of the new slice + a published residual per rank) is staged
    through the host with one all_gather_object per iteration, and the stop test takes the max of the
    published residuals, as peer_sync_stop does."""

    fused = True

    def __init__(self, arrays, rank, world, group=None):
        self.cpu = oracle.Model.from_arrays("port", *arrays)
        self.n = len(arrays[0]) - 1
        self.rank, self.world, self.group = rank, world, group
        self.sb, self.se = sharded.shard_ranges(self.n, world)[rank]

        class M:
            dtype = np.float64
        self.model = M()

    def begin(self, *, initial, frozen=None, rewards=None, discount=0.0, pessimistic=True, maximize=True,
              finite=True, horizon=0, eps=0.0, max_iterations=1_000_000, external_stop=True):
        self.values = [np.asarray(initial, np.float64).copy() for _ in range(2)]
        self.plan = dict(frozen=frozen, rewards=rewards, discount=discount, pess=pessimistic, maxi=maximize,
                         finite=finite, horizon=horizon, eps=eps, max_iterations=max(1, max_iterations))
        self.k = 0
        self.done = False
        self.res_last = 0.0
        dist.barrier(group=self.group)

    def advance(self, iterations):
        for _ in range(iterations):
            if self.done:
                return
            k = self.k + 1
            p = self.plan
            prev = self.values[(k - 1) & 1]
            v, _ = self.cpu.bellman_step(prev, p["pess"], p["maxi"], p["frozen"])
            if p["rewards"] is not None:
                v = p["rewards"] + p["discount"] * v
            mine = v[self.sb:self.se]
            res = float(np.max(np.abs(mine - prev[self.sb:self.se]), initial=0.0))
            got = [None] * self.world
            dist.all_gather_object(got, (self.sb, mine, res), group=self.group)  # the "peer stores"
            out = self.values[k & 1]
            for sb, sl, _ in got:
                out[sb:sb + len(sl)] = sl
            r = max(x[2] for x in got)
            self.k, self.res_last = k, r
            if p["finite"]:
                self.done = k >= p["horizon"]
            elif r <= p["eps"] or k >= p["max_iterations"]:
                self.done = True

    def poll(self):
        return self.k, self.done, self.res_last

    def finish(self):
        k = self.k
        v = self.values[k & 1].copy()
        r = np.abs(v - self.values[(k - 1) & 1]) if k else np.zeros(self.n)
        return {"values": v, "residual": r, "iterations": k}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, arrays, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for plan in cases:
            solver = sharded.ShardedSolver(CpuShard(arrays, rank, world), chunk=5)  # 5: chunks end mid-solve
            try:
                r = solver.solve(**plan)
                out.append((r.values, r.iterations))
            except sharded.NonConvergence as e:
                out.append(("nonconv", e.iterations))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _cases(n):
    goal = np.zeros(n, np.uint8)
    goal[-3:] = 1
    v0 = goal.astype(np.float64)
    rew = np.linspace(0, 1, n)
    return [
        dict(initial=v0, frozen=goal, finite=False, eps=1e-6, pessimistic=True, maximize=True),
        dict(initial=v0, frozen=goal, finite=True, horizon=13, pessimistic=False, maximize=False),
        dict(initial=rew, rewards=rew, discount=0.9, finite=False, eps=1e-7, pessimistic=True, maximize=False),
        dict(initial=v0, frozen=goal, finite=False, eps=1e-14, max_iterations=9, pessimistic=True, maximize=True),
    ]


@pytest.mark.parametrize("world,n", [(2, 37), (3, 37), (4, 9)])
def test_sharded_solve_bit_identical_to_unsharded(world, n):
    """37 states: unequal slices; 9 states over 4 ranks: the last rank owns no state."""
    oracle.build(ref=False)
    arrays = engine.random_imdp(n, 3, 0.25 if n > 20 else 0.5, 0.2, 12)
    cases = _cases(n)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, arrays, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if n == 9:
        assert sharded.shard_ranges(n, world)[-1][0] == sharded.shard_ranges(n, world)[-1][1]
    # unsharded reference: the same loop in one process (world 1)
    cpu = oracle.Model.from_arrays("port", *arrays)
    for i, plan in enumerate(cases):
        v = np.asarray(plan["initial"], np.float64).copy()
        k = 0
        total = plan.get("horizon", 0) if plan["finite"] else plan.get("max_iterations", 1_000_000)
        status = "ok"
        while k < total:
            k += 1
            nv, _ = cpu.bellman_step(v, plan["pessimistic"], plan["maximize"], plan.get("frozen"))
            if plan.get("rewards") is not None:
                nv = plan["rewards"] + plan["discount"] * nv
            res = np.abs(nv - v).max()
            v = nv
            if not plan["finite"] and res <= plan["eps"]:
                break
        else:
            status = "nonconv" if not plan["finite"] else "ok"
        for r in range(world):
            got, iters = results[r][i]
            assert iters == k, (i, r, iters, k)
            if status == "nonconv":
                assert isinstance(got, str) and got == "nonconv"
            else:
                assert np.array_equal(got.view(np.uint64), v.view(np.uint64)), (i, r)
