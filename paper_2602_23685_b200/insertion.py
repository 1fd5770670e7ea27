"""Insertion scoring and repair -- drop-in for the reference's
``vrp_rpd.insertion`` (``/root/reference/pkg/src/vrp_rpd/insertion.py``).

The repair (``reinsert_all``, :484-516, with ``customer_options`` :429-472,
the windowed picks :414-426 and the InsertionContext aggregates :52-350)
runs on the GPU: kernel K5 (csrc/repair.cu), one warp per repair instance,
bit-identical to the reference including its RNG consumption when driven by a
``Generator(Philox)``.  ``reinsert_batch`` repairs many instances per launch
(the ALNS worker batch); ``reinsert_all`` is the reference's one-instance
signature on top of it.

``remove_customers`` (:379-397) and ``removal_gains`` (:538-569) are host
helpers used by the destroy operators (small next to repair).
"""
from __future__ import annotations

import numpy as np
import torch

from . import device as Dev
from . import rng as R
from .schedule import OpKind, Solution

_D, _P = OpKind.DROPOFF, OpKind.PICKUP


class RepairFailed(Exception):
    """No feasible reinsertion exists, or the rebuilt candidate deadlocks."""


class InsertionContext:
    """Mutable set of tours being repaired (the aggregates live on the device
    while a repair runs)."""

    def __init__(self, instance, tours):
        self.instance = instance
        self.tours = [list(t) for t in tours]

    def solution(self) -> Solution:
        return Solution.from_lists(self.tours)


def _pack_tours(tours, n):
    ops = np.full(2 * n, -1, np.int32)
    lens = np.zeros(len(tours), np.int32)
    i = 0
    for v, tour in enumerate(tours):
        for c, kind in tour:
            ops[i] = 2 * (c - 1) + (kind is _P)
            i += 1
        lens[v] = len(tour)
    return ops, lens


def reinsert_batch(instance, partial_ops, partial_lens, removed_lists, regret_ks, gens=None,
                   stream=None):
    """Repair N partial solutions on the GPU.

    partial_ops [N, 2n] / partial_lens [N, m] (numpy or torch), removed_lists:
    N sequences of customers, regret_ks: N ints, gens: N numpy
    Generator(Philox) objects (advanced in place) or None.  Returns numpy
    (ops [N, 2n], lens [N, m], status [N])."""
    Nn = len(removed_lists)
    width = max(1, max((len(r) for r in removed_lists), default=1))
    rem = np.zeros((Nn, width), np.int32)
    nrem = np.zeros(Nn, np.int32)
    for i, r in enumerate(removed_lists):
        rem[i, :len(r)] = r
        nrem[i] = len(r)
    states = None
    if gens is not None:  # one H2D / D2H for all generator states
        gens = [R.as_philox(g) for g in gens]
        states = torch.from_numpy(np.stack([R.state_bytes(g) for g in gens])).to(
            torch.device("cuda", torch.cuda.current_device()))
    out = Dev.repair_batch(instance, partial_ops, partial_lens, rem, nrem,
                           np.asarray(regret_ks, np.int32), states=states, stream=stream)
    if gens is not None:
        host = states.cpu().numpy()
        for i, g in enumerate(gens):
            R.set_state_bytes(g, host[i])
    return out["ops"].cpu().numpy(), out["lens"].cpu().numpy(), out["status"].cpu().numpy()


def reinsert_all(ctx: InsertionContext, removed, regret_k: int = 0, rng=None) -> None:
    """Reinsert every removed customer (greedy when regret_k == 0, else
    regret-k); near-tied choices randomised by ``rng`` (see module doc)."""
    inst = ctx.instance
    ops, lens = _pack_tours(ctx.tours, inst.n)
    gens = None if rng is None else [rng]
    o, l, st = reinsert_batch(inst, ops[None, :], lens[None, :], [list(removed)], [regret_k], gens)
    if st[0] == 1:
        raise RepairFailed("no feasible insertion for some removed customer")
    if st[0] != 0:
        raise ValueError("malformed partial solution")
    ctx.tours = [list(t) for t in Solution.from_arrays(o[0], l[0]).tours]


def _first_capacity_break(tours, k):
    for tour in tours:
        s, lo, hi = 0, 0, k
        for c, kind in tour:
            if kind is _D:
                lo = max(lo, 1 - s)
                s -= 1
            else:
                hi = min(hi, k - 1 - s)
                s += 1
            if lo > hi:
                return c
    return None


def remove_customers(instance, solution: Solution, customers) -> tuple:
    """Drop both ops of `customers`, cascading routes left without a feasible
    initial load (insertion.py:358-397).  Returns (tours, sorted removed)."""
    gone = set(customers)
    tours = [[op for op in tour if op[0] not in gone] for tour in solution.tours]
    while (broken := _first_capacity_break(tours, instance.k)) is not None:
        gone.add(broken)
        tours = [[op for op in tour if op[0] != broken] for tour in tours]
    return tours, sorted(gone)


def _walk_return(seq, d, ready) -> float:
    if not seq:
        return 0.0
    t, loc = 0.0, 0
    for c, kind in seq:
        t += d[loc][c]
        loc = c
        if kind is _P:
            r = ready.get(c)
            if r is not None and r > t:
                t = r
    return t + d[loc][0]


def removal_gains(instance, solution: Solution) -> dict:
    """Makespan reduction estimate per customer under fixed ready times
    (insertion.py:538-569)."""
    d, p = instance.d, instance.p
    tours = [list(t) for t in solution.tours]
    ready = {}
    for tour in tours:
        t, loc = 0.0, 0
        for c, kind in tour:
            t += d[loc][c]
            loc = c
            if kind is _D:
                ready[c] = t + p[c]
    rets = [_walk_return(tour, d, ready) for tour in tours]
    where: dict = {}
    for v, tour in enumerate(tours):
        for c, _ in tour:
            where.setdefault(c, set()).add(v)
    cur = max(rets) if rets else 0.0
    gains = {}
    for c in instance.customers:
        touched = where.get(c, set())
        new_mk = max((r for v, r in enumerate(rets) if v not in touched), default=0.0)
        for v in touched:
            r = _walk_return([op for op in tours[v] if op[0] != c], d, ready)
            if r > new_mk:
                new_mk = r
        gains[c] = cur - new_mk
    return gains
