"""State-sharded value iteration across the GPUs of one box.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the
plumbing).  The IMDP's states are cut into `world` contiguous ranges of equal
length S = ceil(n / world) (state r*S .. r*S+S-1 on rank r): every rank holds
the columns of its own states in HBM and a full replica of the value vector,
padded to world * S entries.  Per iteration k each rank

  1. runs the Bellman kernels for its states (writes V_k[r*S : r*S+S]),
  2. all-gathers the slices in place into its replica of V_k (one
     ncclAllGather of S entries per rank — the only collective),
  3. enqueues the device stop test (solver.hpp:127-134): every rank now holds
     V_k and V_{k-1} in full, so the global residual max |V_k - V_{k-1}| is
     reduced on the device over the whole vector, with no second collective,

all on the shard's CUDA stream, so iterations are enqueued ahead without host
synchronisation; the host polls once per chunk.  Kernels after the stop
iteration are no-ops and the collectives after it re-exchange unchanged
slices, so the result is the stopping iterate on every rank.  Per-state
arithmetic is unchanged by sharding: results are bit-identical to one GPU.

The equal-length cut keeps the exchange a single in-place all-gather; for the
synthetic laws of configs 2-5 it is also nnz-balanced to within a few percent
(reported by ``shard_balance``).  See DESIGN.md "Multi-GPU".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def shard_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """[(state_begin, state_end)] per rank: equal-length contiguous cuts (last may be short or empty)."""
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


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


class DeviceShard:
    """The engine's shard (a DeviceModel built for states [sb, se)) as seen by the driver."""

    def __init__(self, model, rank: int, world: int, n_global: int):
        import torch
        self.torch = torch
        self.model = model
        self.rank, self.world, self.n = rank, world, n_global
        self.S = slice_length(n_global, world)
        self.capacity = self.S * world
        model.set_value_capacity(self.capacity)
        self.device = torch.device("cuda", model.info().device)
        self.stream = torch.cuda.ExternalStream(model.stream(), device=self.device)

    def begin(self, **plan):
        self.model.begin(**plan, external_stop=True)
        t = self.torch
        ts = "<f8" if self.model.dtype == np.float64 else "<f4"
        b0, b1 = self.model.value_buffers()
        self.values = [t.as_tensor(_CudaArray(b, self.capacity, ts), device=self.device) for b in (b0, b1)]
        self.residual = t.as_tensor(_CudaArray(self.model.residual_slots(), 2, "<i8"), device=self.device)

    def advance(self):
        self.model.advance(1)

    def stop_test(self):
        self.model.stop_test()

    def poll(self):
        return self.model.poll()

    def finish(self):
        return self.model.finish()

    def stream_context(self):
        return self.torch.cuda.stream(self.stream)


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
    """Drives one rank's shard through a sharded solve (the loop of
    detail::iterate, solver.hpp:85-137, with the exchange step added)."""

    def __init__(self, shard, group=None, chunk: int = 32):
        import torch.distributed as dist
        self.dist = dist
        self.shard = shard
        self.group = group
        self.chunk = chunk

    def _exchange(self, k: int):
        sh, dist = self.shard, self.dist
        buf = sh.values[k & 1]
        r, S = sh.rank, sh.S
        dist.all_gather_into_tensor(buf, buf[r * S:(r + 1) * S], group=self.group)

    def enqueue(self, k: int):
        """Iteration k: local kernels, exchange, stop test — all stream-ordered."""
        self.shard.advance()
        self._exchange(k)
        self.shard.stop_test()

    def solve(self, *, finite: bool, horizon: int = 0, max_iterations: int = 1_000_000, eps: float = 0.0,
              **plan) -> ShardedResult:
        sh = self.shard
        total = horizon if finite else max_iterations
        sh.begin(finite=finite, horizon=horizon, max_iterations=max_iterations, eps=eps, **plan)
        k = 0
        done = False
        res = 0.0
        with sh.stream_context():
            while k < total and not done:
                for _ in range(min(self.chunk, total - k)):
                    k += 1
                    self.enqueue(k)
                _, done, res = sh.poll()
        out = sh.finish()
        iters = out["iterations"]
        if not finite and iters > 0 and not res <= np.dtype(sh.model.dtype).type(eps):
            raise NonConvergence(iters, res)
        return ShardedResult(out["values"][:sh.n], out["residual"][:sh.n], iters, True)

