"""Problem specifications and the solve entry points, over the device engine.

Python mirror of the reference's problem half of the API, for tests, the
benchmark and the sharded driver:

  property structs / Specification / check_property   property.hpp:14-180
  detail::make_plan                                    solver.hpp:40-80
  value_iteration / control_synthesis / verify_policy  solver.hpp:149-251
  bellman_step                                         bellman.hpp:127-133

Error behaviour follows the reference exception types (errors.hpp:11-140);
the iteration itself always runs on the GPU through the C ABI.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .engine import (ERR_INFEASIBLE_COLUMN, ERR_NON_CONVERGENCE, DeviceModel, EngineError)


class Error(RuntimeError):
    pass


class ModelError(Error):
    def __init__(self, message, column=-1):
        super().__init__(message)
        self.column = column


class NonConvergence(Error):
    def __init__(self, iterations, residual):
        super().__init__(f"no convergence after {iterations} iterations (max residual {residual:f})")
        self.iterations = iterations
        self.residual = residual


class PropertyStateOutOfRange(Error):
    def __init__(self, state, n):
        super().__init__(f"property state index {state} out of range (model has {n} states)")


class InvalidProperty(Error):
    def __init__(self, msg):
        super().__init__("invalid property: " + msg)


class InvalidPolicyAction(Error):
    def __init__(self, msg):
        super().__init__("invalid policy: " + msg)


PESSIMISTIC, OPTIMISTIC = "pessimistic", "optimistic"
MINIMIZE, MAXIMIZE = "minimize", "maximize"


@dataclass
class FiniteTimeReachability:
    goal: list
    horizon: int


@dataclass
class InfiniteTimeReachability:
    goal: list
    eps: float


@dataclass
class FiniteTimeReachAvoid:
    reach: list
    avoid: list
    horizon: int


@dataclass
class InfiniteTimeReachAvoid:
    reach: list
    avoid: list
    eps: float


@dataclass
class FiniteTimeReward:
    rewards: np.ndarray
    discount: float
    horizon: int


@dataclass
class InfiniteTimeReward:
    rewards: np.ndarray
    discount: float
    eps: float


@dataclass
class Specification:
    property: object
    satisfaction: str = PESSIMISTIC
    strategy: str = MAXIMIZE


@dataclass
class Plan:
    initial: np.ndarray
    frozen: np.ndarray | None
    finite: bool
    horizon: int = 0
    eps: float = 0.0
    rewards: np.ndarray | None = None
    discount: float = 0.0


@dataclass
class ValueFunction:
    values: np.ndarray
    iterations: int
    residual: np.ndarray

    def max_residual(self):
        return self.residual.max(initial=0)


@dataclass
class Policy:
    """Stationary: columns[n]; time-dependent: columns[n, horizon] (entry (s, t))."""
    columns: np.ndarray
    time_dependent: bool = False
    labels: list = field(default_factory=list)


def _check_states(states, n):
    for s in states:
        if s < 0 or s >= n:
            raise PropertyStateOutOfRange(s, n)


def check_property(p, n: int) -> None:
    """property.hpp:132-180."""
    if isinstance(p, (FiniteTimeReachability, InfiniteTimeReachability)):
        _check_states(p.goal, n)
    elif isinstance(p, (FiniteTimeReachAvoid, InfiniteTimeReachAvoid)):
        _check_states(p.reach, n)
        _check_states(p.avoid, n)
        for r in p.reach:
            if r in set(p.avoid):
                raise InvalidProperty(f"reach and avoid sets overlap at state {r}")
    else:
        if len(p.rewards) != n:
            raise InvalidProperty(f"reward vector length {len(p.rewards)} does not match {n} states")
        if p.discount < 0 or p.discount > 1:
            raise InvalidProperty("discount must be in [0,1]")
    if hasattr(p, "horizon"):
        if p.horizon < 0:
            raise InvalidProperty("time horizon must be non-negative")
    else:
        if not p.eps > 0:
            raise InvalidProperty("eps must be positive")
        if isinstance(p, InfiniteTimeReward) and p.discount >= 1:
            raise InvalidProperty("infinite-time reward requires discount < 1")


def make_plan(spec: Specification, n: int, dtype) -> Plan:
    """solver.hpp:40-80."""
    p = spec.property
    check_property(p, n)
    dtype = np.dtype(dtype)
    v0 = np.zeros(n, dtype)
    frozen = np.zeros(n, np.uint8)
    rewards = None
    discount = 0.0
    if isinstance(p, (FiniteTimeReachability, InfiniteTimeReachability)):
        v0[list(p.goal)] = 1
        frozen[list(p.goal)] = 1
    elif isinstance(p, (FiniteTimeReachAvoid, InfiniteTimeReachAvoid)):
        v0[list(p.reach)] = 1
        frozen[list(p.reach)] = 1
        frozen[list(p.avoid)] = 1
    else:
        rewards = np.ascontiguousarray(p.rewards, dtype)
        v0 = rewards.copy()
        discount = float(dtype.type(p.discount))
        frozen = None
    finite = hasattr(p, "horizon")
    return Plan(v0, frozen, finite, horizon=getattr(p, "horizon", 0), eps=getattr(p, "eps", 0.0),
                rewards=rewards, discount=discount)


def _kw(spec: Specification, plan: Plan, max_iterations: int):
    return dict(initial=plan.initial, frozen=plan.frozen, finite=plan.finite, horizon=plan.horizon,
                eps=float(np.dtype(plan.initial.dtype).type(plan.eps)), rewards=plan.rewards,
                discount=plan.discount, pessimistic=spec.satisfaction == PESSIMISTIC,
                maximize=spec.strategy == MAXIMIZE, max_iterations=max_iterations)


def _translate(e: EngineError):
    if e.status == ERR_INFEASIBLE_COLUMN:
        return ModelError(e.message, e.column)
    if e.status == ERR_NON_CONVERGENCE:
        return NonConvergence(e.iterations, e.residual)
    return e


def _run(model: DeviceModel, kw, **extra):
    try:
        return model.solve(**kw, **extra)
    except EngineError as e:
        raise _translate(e) from None


def value_iteration(model: DeviceModel, spec: Specification, max_iterations=1_000_000, on_iteration=None):
    plan = make_plan(spec, model.num_states, model.dtype)
    out = _run(model, _kw(spec, plan, max_iterations), on_iteration=on_iteration)
    return ValueFunction(out["values"], out["iterations"], out["residual"])


def control_synthesis(model: DeviceModel, spec: Specification, stateptr, max_iterations=1_000_000):
    """Frozen states are assigned their first column (solver.hpp:170-172)."""
    plan = make_plan(spec, model.num_states, model.dtype)
    stateptr = np.asarray(stateptr)
    first = stateptr[:-1].astype(np.int32)
    if plan.finite:
        out = _run(model, _kw(spec, plan, max_iterations), record="all")
        ch = out["chosen"]  # [horizon][n], row t
        cols = np.where(ch >= 0, ch, first[None, :]).T.copy() if plan.horizon > 0 else np.zeros((len(first), 0), np.int32)
        policy = Policy(cols, True)
    else:
        out = _run(model, _kw(spec, plan, max_iterations), record="last")
        policy = Policy(np.where(out["chosen"] >= 0, out["chosen"], first), False)
    return policy, ValueFunction(out["values"], out["iterations"], out["residual"])


def verify_policy(model: DeviceModel, policy: Policy, spec: Specification, stateptr, max_iterations=1_000_000):
    """solver.hpp:204-251, with the policy given as column indices."""
    n = model.num_states
    plan = make_plan(spec, n, model.dtype)
    stateptr = np.asarray(stateptr)
    cols = np.asarray(policy.columns, np.int32)
    if policy.time_dependent:
        if not plan.finite:
            raise InvalidPolicyAction("a time-dependent policy cannot be evaluated against an infinite-time property")
        if cols.shape != (n, plan.horizon):
            raise InvalidPolicyAction(f"policy shape {cols.shape[0]}x{cols.shape[1] if cols.ndim > 1 else 0} "
                                      f"does not match {n} states, horizon {plan.horizon}")
        forced = cols.T.copy()  # row t
    else:
        if len(cols) != n:
            raise InvalidPolicyAction(f"stationary policy has {len(cols)} entries for {n} states")
        forced = cols
    lo, hi = stateptr[:-1], stateptr[1:]
    bad = (forced < lo) | (forced >= hi)
    if bad.any():
        s = int(np.argwhere(bad)[0][-1])
        raise InvalidPolicyAction(f"state {s} has no action column {int(forced.reshape(-1, n)[0][s])}")
    kw = _kw(spec, plan, max_iterations)
    kw["forced"] = forced
    out = _run(model, kw)
    return ValueFunction(out["values"], out["iterations"], out["residual"])


def bellman_step(model: DeviceModel, values, satisfaction=PESSIMISTIC, strategy=MAXIMIZE, frozen=None):
    try:
        return model.bellman_step(values, satisfaction == PESSIMISTIC, strategy == MAXIMIZE, frozen)
    except EngineError as e:
        raise _translate(e) from None
