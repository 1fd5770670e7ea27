"""Deterministic input generators shared by make_golden.py and the tests.

Everything here is numpy-only (no reference import), keyed by Philox keys,
so the GPU box regenerates the exact inputs the golden outputs were made from.
Each golden record also stores a sha256 of its inputs, so drift is caught.
"""
from __future__ import annotations

import hashlib

import numpy as np


def philox(*key) -> np.random.Generator:
    """Generator(Philox(key=(k0, k1))); a third component is folded into k1."""
    k = [int(x) for x in key]
    if len(k) == 3:
        k = [k[0], (k[1] << 32) | k[2]]
    return np.random.Generator(np.random.Philox(key=tuple(k)))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def chromosomes(n: int, count: int, key) -> np.ndarray:
    """Uniform random keys, like brkga.random_population (brkga.py:78-79)."""
    return philox(*key).random((count, 4 * n))


def random_candidates(n: int, m: int, count: int, key):
    """Structurally valid, possibly infeasible candidates in the spirit of
    pkg/tests/conftest.py:24-30: a random op order, each op to a random vehicle.
    Returns (ops int32 [count, 2n] vehicle-major, lens int32 [count, m])."""
    g = philox(*key)
    ops = np.empty((count, 2 * n), np.int32)
    lens = np.empty((count, m), np.int32)
    for i in range(count):
        order = g.permutation(2 * n).astype(np.int32)
        veh = g.integers(m, size=2 * n)
        stable = np.argsort(veh, kind="stable")
        ops[i] = order[stable]
        lens[i] = np.bincount(veh, minlength=m)
    return ops, lens


def block_candidates(n: int, m: int, k: int, count: int, key):
    """Feasible-by-construction candidates: per route, blocks of <= k dropoffs
    followed by their own pickups (test_schedule.py:241-257 structure)."""
    g = philox(*key)
    ops = np.empty((count, 2 * n), np.int32)
    lens = np.empty((count, m), np.int32)
    for i in range(count):
        cust = g.permutation(n) + 1
        routes = [[] for _ in range(m)]
        pos = 0
        while pos < n:
            v = int(g.integers(m))
            blk = cust[pos:pos + int(g.integers(1, k + 1))]
            pos += len(blk)
            routes[v] += [2 * (c - 1) for c in blk]
            routes[v] += [2 * (c - 1) + 1 for c in blk]
        flat = np.concatenate([np.asarray(r, np.int32) for r in routes]) if n else np.zeros(0, np.int32)
        ops[i] = flat
        lens[i] = [len(r) for r in routes]
    return ops, lens


def swap_perturb(ops, lens, key, swaps: int = 2):
    """Swap random adjacent ops inside routes (creates deadlocks/capacity breaks)."""
    g = philox(*key)
    ops = ops.copy()
    for i in range(ops.shape[0]):
        off = np.concatenate([[0], np.cumsum(lens[i])])
        for _ in range(swaps):
            v = int(g.integers(lens.shape[1]))
            L = int(lens[i, v])
            if L < 2:
                continue
            j = int(g.integers(L - 1)) + int(off[v])
            ops[i, j], ops[i, j + 1] = ops[i, j + 1], ops[i, j]
    return ops


def arrays_to_lists(ops_row, lens_row):
    """Vehicle-major op codes -> [[(c, 'D'|'P'), ...], ...]."""
    tours, at = [], 0
    for L in lens_row:
        seg = ops_row[at:at + int(L)]
        at += int(L)
        tours.append([(int(o) // 2 + 1, "P" if int(o) & 1 else "D") for o in seg])
    return tours


def lists_to_arrays(tours, n):
    ops = np.full(2 * n, -1, np.int32)
    lens = np.zeros(len(tours), np.int32)
    at = 0
    for v, tour in enumerate(tours):
        for c, kind in tour:
            k = kind if isinstance(kind, str) else kind.value
            ops[at] = 2 * (int(c) - 1) + (1 if k == "P" else 0)
            at += 1
        lens[v] = len(tour)
    return ops, lens
