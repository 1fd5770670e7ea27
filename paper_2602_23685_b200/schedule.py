"""Solution model and makespan evaluation -- drop-in for the reference's
``vrp_rpd.schedule`` (``/root/reference/pkg/src/vrp_rpd/schedule.py``).

The data model (``OpKind``, ``Solution``, ``Event``, ``Schedule``, the
``ScheduleError`` family) keeps the reference's names and fields.  The
evaluators run on the GPU through the C-ABI (``device.makespan_batch`` /
``device.evaluate_records``, kernels K1/K2 in ``csrc/makespan.cu``); a
per-candidate status code is turned back into the reference's exception:

  exact_makespan     schedule.py:265-316   K1, mode EXACT (no structural check)
  evaluate           schedule.py:188-257   K1, mode EVALUATE + event records
  two_pass_estimate  schedule.py:345-393   K2

``*_batch`` variants score many candidates per launch and are the intended
hot-path API.  ``validate_solution``, ``route_initial_load`` and
``coordination_metrics`` are host helpers kept for API parity; they are not
on the scoring path.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

import numpy as np

from . import _native as N


class OpKind(Enum):
    DROPOFF = "D"
    PICKUP = "P"


class ScheduleError(Exception):
    """Base class for evaluation failures."""


class MalformedSolution(ScheduleError):
    """Not exactly one dropoff and one pickup per customer."""


class CapacityViolation(ScheduleError):
    """No initial load in [0, k] lets some route execute."""


class Deadlock(ScheduleError):
    """Circular cross-vehicle waits."""


_STATUS_ERRORS = {N.VRP_CAPACITY: (CapacityViolation, "no feasible initial load for a route"),
                  N.VRP_DEADLOCK: (Deadlock, "circular cross-vehicle waits"),
                  N.VRP_MALFORMED: (MalformedSolution, "solution breaks the one-D/one-P structure")}


def raise_for_status(status: int) -> None:
    if status != N.VRP_OK:
        cls, msg = _STATUS_ERRORS[int(status)]
        raise cls(msg)


@dataclass(frozen=True)
class Solution:
    """Per-vehicle ordered tours of (customer, OpKind) pairs."""

    tours: tuple

    @classmethod
    def from_lists(cls, tours) -> "Solution":
        return cls(tuple(tuple((c, kind if isinstance(kind, OpKind) else OpKind(kind))
                               for c, kind in tour) for tour in tours))

    def to_lists(self):
        return [list(tour) for tour in self.tours]

    def to_dict(self, instance_label: str = "") -> dict:
        return {"instance_label": instance_label,
                "tours": [[[c, kind.value] for c, kind in tour] for tour in self.tours]}

    @classmethod
    def from_dict(cls, doc: dict) -> "Solution":
        return cls.from_lists([[(int(c), OpKind(k)) for c, k in tour] for tour in doc["tours"]])

    def save(self, path, instance_label: str = "") -> None:
        Path(path).write_text(json.dumps(self.to_dict(instance_label)), encoding="utf-8")

    @classmethod
    def load(cls, path) -> "Solution":
        return cls.from_dict(json.loads(Path(path).read_text(encoding="utf-8")))

    # -- device layout ------------------------------------------------------
    def to_arrays(self, n: int):
        """(ops int32 [max(2n, #ops)], lens int32 [len(tours)]) with op code
        2(c-1)+kind; customers outside 1..n encode as -1 (MALFORMED on device)."""
        total = sum(len(t) for t in self.tours)
        ops = np.full(max(2 * n, total), -1, dtype=np.int32)
        lens = np.fromiter((len(t) for t in self.tours), dtype=np.int32, count=len(self.tours))
        i = 0
        for tour in self.tours:
            for c, kind in tour:
                ops[i] = 2 * (c - 1) + (kind is OpKind.PICKUP) if 1 <= c <= n else -1
                i += 1
        return ops, lens

    @classmethod
    def from_arrays(cls, ops, lens) -> "Solution":
        ops = np.asarray(ops)
        tours, at = [], 0
        for L in np.asarray(lens).tolist():
            seg = ops[at:at + L].tolist()
            at += L
            tours.append(tuple((o // 2 + 1, OpKind.PICKUP if o & 1 else OpKind.DROPOFF)
                               for o in seg))
        return cls(tuple(tours))


@dataclass
class Event:
    customer: int
    kind: OpKind
    arrival: float
    time: float
    q_after: int


@dataclass
class Schedule:
    t_drop: dict
    t_pickup: dict
    drop_vehicle: dict
    pickup_vehicle: dict
    returns: list
    makespan: float
    events: list
    initial_loads: list

    def bottleneck(self) -> int:
        """First vehicle with the largest return (schedule.py:105-110)."""
        top = max(self.returns) if self.returns else 0.0
        for v, r in enumerate(self.returns):
            if r == top:
                return v
        return 0

    def to_rows(self) -> list:
        return [{"vehicle": v, "seq": i, "customer": e.customer, "op": e.kind.value,
                 "arrival": e.arrival, "time": e.time, "q_after": e.q_after}
                for v, evs in enumerate(self.events) for i, e in enumerate(evs)]


@dataclass(frozen=True)
class CoordinationMetrics:
    cross_agent_pct: float
    interleaved_pct: float


# --------------------------------------------------------------------------
# host helpers kept for API parity
# --------------------------------------------------------------------------

def validate_solution(instance, solution: Solution) -> None:
    """MalformedSolution unless every customer has exactly one D and one P."""
    if len(solution.tours) != instance.m:
        raise MalformedSolution(f"solution has {len(solution.tours)} tours for {instance.m} vehicles")
    seen = {OpKind.DROPOFF: set(), OpKind.PICKUP: set()}
    for tour in solution.tours:
        for c, kind in tour:
            if not 1 <= c <= instance.n:
                raise MalformedSolution(f"unknown customer {c}")
            if c in seen[kind]:
                raise MalformedSolution(f"customer {c} has duplicate {kind.value}")
            seen[kind].add(c)
    every = set(instance.customers)
    if seen[OpKind.DROPOFF] != every or seen[OpKind.PICKUP] != every:
        raise MalformedSolution("missing dropoffs or pickups")


def route_initial_load(tour, k: int) -> int:
    """Smallest feasible initial load of one route (schedule.py:159-185)."""
    s, lo, hi = 0, 0, k
    for c, kind in tour:
        if kind is OpKind.DROPOFF:
            lo = max(lo, 1 - s)
            s -= 1
        else:
            hi = min(hi, k - 1 - s)
            s += 1
        if lo > hi:
            raise CapacityViolation(f"route infeasible at customer {c} for capacity {k}")
    return lo


def makespan(schedule: Schedule) -> float:
    return max(schedule.returns) if schedule.returns else 0.0


def coordination_metrics(instance, solution: Solution, schedule: Schedule) -> CoordinationMetrics:
    """Cross-agent / interleaved percentages of a realised schedule."""
    n = instance.n
    cross = sum(schedule.drop_vehicle[c] != schedule.pickup_vehicle[c] for c in instance.customers)
    inter = 0
    for c in instance.customers:
        a, b = schedule.t_drop[c], schedule.t_pickup[c]
        owners = {schedule.drop_vehicle[c], schedule.pickup_vehicle[c]}
        if any(e.customer != c and a < e.time < b for v in owners for e in schedule.events[v]):
            inter += 1
    return CoordinationMetrics(cross_agent_pct=100.0 * cross / n, interleaved_pct=100.0 * inter / n)


# --------------------------------------------------------------------------
# device evaluators
# --------------------------------------------------------------------------

def _one(instance, solution: Solution, mode: int) -> float:
    if len(solution.tours) != instance.m:
        if mode == N.MODE_EXACT:
            raise ValueError(f"solution has {len(solution.tours)} tours for {instance.m} vehicles")
        raise MalformedSolution(f"solution has {len(solution.tours)} tours for {instance.m} vehicles")
    from .device import makespan_batch
    ops, lens = solution.to_arrays(instance.n)
    res = makespan_batch(instance, ops[None, :], lens[None, :], mode=mode)
    status = int(res["status"].item())
    raise_for_status(status)
    return float(res["z"].item())


def exact_makespan(instance, solution: Solution) -> float:
    """Makespan under evaluate's semantics without records (K1, GPU)."""
    return _one(instance, solution, N.MODE_EXACT)


def two_pass_estimate(instance, solution: Solution) -> float:
    """Two-pass makespan estimate (K2, GPU)."""
    return _one(instance, solution, N.MODE_TWO_PASS)


def evaluate(instance, solution: Solution) -> Schedule:
    """Exact event-driven evaluation with full records (K1 + records, GPU)."""
    if len(solution.tours) != instance.m:
        raise MalformedSolution(f"solution has {len(solution.tours)} tours for {instance.m} vehicles")
    from .device import evaluate_records
    ops, lens = solution.to_arrays(instance.n)
    res = evaluate_records(instance, ops[None, :], lens[None, :])
    status = int(res["status"].item())
    raise_for_status(status)
    arrival = res["arrival"][0].cpu().numpy()
    times = res["time"][0].cpu().numpy()
    q0 = [int(x) for x in res["q0"][0].cpu().tolist()]
    returns = [float(x) for x in res["returns"][0].cpu().tolist()]
    t_drop, t_pick, dveh, pveh = {}, {}, {}, {}
    events = []
    i = 0
    for v, tour in enumerate(solution.tours):
        q = q0[v]
        evs = []
        for c, kind in tour:
            a, t = float(arrival[i]), float(times[i])
            if kind is OpKind.DROPOFF:
                q -= 1
                t_drop[c], dveh[c] = t, v
            else:
                q += 1
                t_pick[c], pveh[c] = t, v
            evs.append(Event(c, kind, a, t, q))
            i += 1
        events.append(evs)
    return Schedule(t_drop=t_drop, t_pickup=t_pick, drop_vehicle=dveh, pickup_vehicle=pveh,
                    returns=returns, makespan=max(returns) if returns else 0.0, events=events,
                    initial_loads=q0)


def pack_solutions(instance, solutions, op_dtype=np.int32):
    """List of Solution -> (ops [N, 2n], lens [N, m]) numpy arrays."""
    n, m = instance.n, instance.m
    ops = np.full((len(solutions), 2 * n), -1, dtype=op_dtype)
    lens = np.zeros((len(solutions), m), dtype=np.int32)
    for i, sol in enumerate(solutions):
        o, l = sol.to_arrays(n)
        if len(l) != m or len(o) > 2 * n:
            raise MalformedSolution("solution does not fit the instance")
        ops[i], lens[i] = o, l
    return ops, lens


def score_host_batch(instance, ops, lens, mode: int = N.MODE_EXACT, chunk: int = 1 << 14):
    """Host candidates in, host (z, status) out; pipelined H2D / K1 / D2H."""
    from .device import score_host_batch as _s
    return _s(instance, ops, lens, mode=mode, chunk=chunk)


def exact_makespan_batch(instance, ops, lens, mode: int = N.MODE_EXACT, stream=None):
    """Device batch scoring; returns (z, status) as torch tensors on the GPU."""
    from .device import makespan_batch
    r = makespan_batch(instance, ops, lens, mode=mode, stream=stream)
    return r["z"], r["status"]
