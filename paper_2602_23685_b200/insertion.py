"""Insertion scoring and repair -- drop-in for the reference's
``vrp_rpd.insertion`` (``/root/reference/pkg/src/vrp_rpd/insertion.py``).

The repair (``reinsert_all``, :484-516, with ``customer_options`` :429-472,
the windowed picks :414-426 and the InsertionContext aggregates :52-350)
runs on the GPU: kernel K5 (csrc/repair.cu), one warp per repair instance,
bit-identical to the reference including its RNG consumption when driven by a
``Generator(Philox)``.  ``reinsert_batch`` repairs many instances per launch
(the ALNS worker batch); ``reinsert_all`` is the reference's one-instance
signature on top of it.

``remove_customers`` (:379-397) and ``removal_gains`` (:538-569) run K6's
device code (``vrp_remove_batch`` / ``vrp_removal_gains``) on one solution.
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


def remove_customers(instance, solution: Solution, customers) -> tuple:
    """Drop both operations of ``customers`` and cascade every customer whose
    removal leaves a route without a feasible initial load
    (insertion.py:379-397).  Runs K6's removal on the device
    (vrp_remove_batch, batch of one).  Returns (tours, sorted removed)."""
    n = instance.n
    ops, lens = solution.to_arrays(n)
    picked = np.asarray(sorted({int(c) for c in customers}), np.int32)
    if picked.size == 0:
        picked = np.zeros(1, np.int32)
        count = 0
    else:
        count = picked.size
    r = Dev.remove_batch(instance, ops[None, :2 * n], lens[None], picked[None], np.array([count], np.int32))
    o, ln = r["ops"][0].cpu().numpy(), r["lens"][0].cpu().numpy()
    nr = int(r["nremoved"][0].item())
    removed = [int(c) for c in r["removed"][0, :nr].cpu().numpy()]
    return [list(t) for t in Solution.from_arrays(o, ln).tours], removed


def removal_gains(instance, solution: Solution) -> dict:
    """Estimated makespan reduction of removing each customer, ready times
    held fixed (insertion.py:538-569), on the device (vrp_removal_gains)."""
    ops, lens = solution.to_arrays(instance.n)
    g = Dev.removal_gains_batch(instance, ops[None, :2 * instance.n], lens[None])[0].cpu().numpy()
    return {c: float(g[c]) for c in instance.customers}
