"""State-sharded value iteration across the GPUs of one box, one process per GPU.

The IMDP's states are cut into `world` contiguous ranges (``shard_ranges``);
every rank holds the columns of its own states in HBM and a full replica of
the value vector.  Per iteration k each rank runs the Bellman kernels for its
states, and the exchange is fused into them:

  * the action kernel stores every new value V_k[s] of the rank's states into
    every peer's V_k buffer over NVLink (peer memory mapped with CUDA IPC) as
    it computes it — the transfer overlaps the computation of the local rows
    by construction, there is no separate collective;
  * its last block publishes the rank's residual and the iteration number to
    every peer (system-scope release);
  * a one-warp kernel (peer_sync_stop) waits for every rank's flag of
    iteration k (acquire) and runs the stop test (solver.hpp:127-134) on the
    maximum published residual — the same numbers, so the same decision, on
    every rank.

All of it is stream-ordered on the shard's CUDA stream, so iterations are
enqueued ahead without host synchronisation; the host polls once per chunk.
Kernels after the stop iteration are no-ops on every rank.  Per-state
arithmetic is unchanged by sharding: results are bit-identical to one GPU.

``torch.distributed`` is plumbing only: the 64-byte IPC handles of the
exchange windows are swapped once with ``all_gather_object`` and every
solve's begin is followed by one barrier (begin resets the windows).

``NcclShard`` keeps the unfused baseline for comparison: local kernels, then
an in-place ``all_gather`` of the padded V slices with NCCL, then a device
stop test over the gathered vector — three steps per iteration on one stream.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def shard_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """[(state_begin, state_end)] per rank: equal-length contiguous cuts (the last may be short or empty)."""
    if n < 0 or world < 1:
        raise ValueError("bad sizes")
    S = max(1, math.ceil(n / world))
    return [(min(n, r * S), min(n, (r + 1) * S)) for r in range(world)]


def slice_length(n: int, world: int) -> int:
    return max(1, math.ceil(n / world))


def shard_balance(state_nnz: np.ndarray, world: int) -> float:
    """max over ranks of shard transitions / mean (1.0 = perfectly balanced)."""
    tot = []
    for sb, se in shard_ranges(len(state_nnz), world):
        tot.append(int(np.sum(state_nnz[sb:se])))
    mean = sum(tot) / world
    return max(tot) / mean if mean else 1.0


def slice_csc(stateptr, colptr, rowval, lower, upper, sb: int, se: int):
    """Local CSC arrays of states [sb, se): stateptr/colptr rebased, rows kept global."""
    stateptr = np.asarray(stateptr)
    colptr = np.asarray(colptr)
    cb, ce = int(stateptr[sb]), int(stateptr[se])
    b, e = int(colptr[cb]), int(colptr[ce])
    return (stateptr[sb:se + 1] - cb, colptr[cb:ce + 1] - b, rowval[b:e], lower[b:e], upper[b:e])


class PeerShard:
    """The engine's shard (a DeviceModel built for states [sb, se)) connected to its peers' exchange
    windows: one collective at construction (the IPC handles), none per iteration."""

    fused = True

    def __init__(self, model, rank: int, world: int, n_global: int, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.model = model
        self.rank, self.world, self.n = rank, world, n_global
        model.set_value_capacity(n_global)
        handles = [None] * world
        dist.all_gather_object(handles, model.exchange_export(), group=group)
        model.exchange_connect(rank, world, handles)

    def begin(self, **plan):
        self.model.begin(**plan, external_stop=True)
        self.dist.barrier(group=self.group)  # every window is reset before any rank publishes iteration 1

    def advance(self, iterations: int):
        self.model.advance(iterations)       # kernels + peer stores + peer_sync_stop, per iteration

    def poll(self):
        return self.model.poll()

    def finish(self):
        return self.model.finish()


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


class NcclShard:
    """Unfused baseline: V padded to world equal slices, one in-place NCCL all-gather and a device stop test
    over the gathered vector after each iteration's kernels."""

    fused = False

    def __init__(self, model, rank: int, world: int, n_global: int, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.model = model
        self.rank, self.world, self.n = rank, world, n_global
        self.S = slice_length(n_global, world)
        if shard_ranges(n_global, world)[rank][0] != min(n_global, rank * self.S):
            raise ValueError("the NCCL baseline needs equal-length slices (shard_ranges)")
        self.capacity = self.S * world
        model.set_value_capacity(self.capacity)
        self.device = torch.device("cuda", model.info().device)
        self.stream = torch.cuda.ExternalStream(model.stream(), device=self.device)

    def begin(self, **plan):
        self.model.begin(**plan, external_stop=True)
        ts = "<f8" if self.model.dtype == np.float64 else "<f4"
        b0, b1 = self.model.value_buffers()
        self.values = [self.torch.as_tensor(_CudaArray(b, self.capacity, ts), device=self.device) for b in (b0, b1)]
        self.k = 0

    def advance(self, iterations: int):
        with self.torch.cuda.stream(self.stream):
            for _ in range(iterations):
                self.k += 1
                self.model.advance(1)
                buf = self.values[self.k & 1]
                r, S = self.rank, self.S
                self.dist.all_gather_into_tensor(buf, buf[r * S:(r + 1) * S], group=self.group)
                self.model.stop_test()

    def poll(self):
        return self.model.poll()

    def finish(self):
        return self.model.finish()


@dataclass
class ShardedResult:
    values: np.ndarray
    residual: np.ndarray
    iterations: int
    converged: bool   # finite: horizon reached; infinite: max residual <= eps


class NonConvergence(RuntimeError):
    """Infinite horizon: the iteration cap was reached (solver.hpp:131-133)."""

    def __init__(self, iterations, residual):
        super().__init__(f"no convergence after {iterations} iterations (max residual {residual:f})")
        self.iterations = iterations
        self.residual = residual


class ShardedSolver:
    """Drives one rank's shard through a sharded solve (the loop of detail::iterate, solver.hpp:85-137,
    with the exchange fused into the iteration)."""

    def __init__(self, shard, group=None, chunk: int = 64):
        self.shard = shard
        self.group = group
        self.chunk = chunk

    def solve(self, *, finite: bool, horizon: int = 0, max_iterations: int = 1_000_000, eps: float = 0.0,
              **plan) -> ShardedResult:
        sh = self.shard
        total = horizon if finite else max(1, max_iterations)  # iterate() always runs step 1
        sh.begin(finite=finite, horizon=horizon, max_iterations=max_iterations, eps=eps, **plan)
        launched, done, res = 0, False, 0.0
        step, last = 4, None
        while launched < total and not done:
            n = min(step, total - launched)
            sh.advance(n)
            launched += n
            k, done, res = sh.poll()
            # geometric residual decay near convergence: enqueue about as many as the stop test needs
            if not finite and last and 0 < res < last[1] and k > last[0] and eps > 0:
                rate = math.log(res / last[1]) / (k - last[0])
                need = math.log(eps / res) / rate
                step = max(1, min(int(need) + 1, self.chunk)) if math.isfinite(need) else min(2 * step, self.chunk)
            else:
                step = min(2 * step, self.chunk)
            last = (k, res)
        out = sh.finish()
        iters = out["iterations"]
        dt = getattr(getattr(sh, "model", None), "dtype", np.float64)
        if not finite and not res <= np.dtype(dt).type(eps):
            raise NonConvergence(iters, res)
        return ShardedResult(out["values"][:sh.n], out["residual"][:sh.n], iters, True)
