"""CPU restatement of the reference's destroy side of ALNS -- TEST
INFRASTRUCTURE ONLY (imported by ``tests/``; never by the product package).

Restates, on flat (ops, lens) arrays:
  removal_gains      ref insertion.py:522-569 (fixed ready times, walk per route)
  destroy            ref alns.py:167-251 (six operators; Fisher-Yates sample,
                     power-law pick, Shaw relatedness alns.py:145-155)
  remove_customers   ref insertion.py:358-397 -- the C oracle's
                     ``oracle.remove_customers``
The schedule the Shaw / critical-path operators read comes from the C
oracle's evaluate (``oracle.evaluate_one``).  The generator must be a
``Generator(Philox)`` (or any numpy Generator): every draw is made with the
reference's call in the reference's order.

Pinned by tests/test_host_alns.py against the reference's destroy goldens.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

SHAW_W_TRAVEL, SHAW_W_TIME, SHAW_W_AGENT = 9.0, 3.0, 5.0  # ref alns.py:31-33
WORST_POWER = 6.0  # ref alns.py:34


def _routes(ops, lens):
    out, at = [], 0
    for L in np.asarray(lens).tolist():
        out.append([int(x) for x in np.asarray(ops)[at:at + L]])
        at += L
    return out


def removal_bounds(n: int):
    q_max = max(4, n // 20)
    return max(4, q_max // 2), q_max  # ref alns.py:102-109


def removal_gains(inst, ops, lens) -> np.ndarray:
    """gains[c] for c = 1..n (index 0 unused): current makespan minus the
    makespan with c's two ops removed, every pickup's ready time held at its
    dropoff's no-wait time + p (ref insertion.py:538-569)."""
    d, p = inst.arrays()
    routes = _routes(ops, lens)
    ready = {}
    for r in routes:
        t, loc = 0.0, 0
        for op in r:
            c = op // 2 + 1
            t += d[loc][c]
            loc = c
            if not op & 1:
                ready[c] = t + p[c]

    def walk(seq):
        if not seq:
            return 0.0
        t, loc = 0.0, 0
        for op in seq:
            c = op // 2 + 1
            t += d[loc][c]
            loc = c
            if op & 1:
                rd = ready.get(c)
                if rd is not None and rd > t:
                    t = rd
        return t + d[loc][0]

    rets = [walk(r) for r in routes]
    cur = max(rets) if rets else 0.0
    on = {}
    for v, r in enumerate(routes):
        for op in r:
            on.setdefault(op // 2 + 1, set()).add(v)
    gains = np.zeros(inst.n + 1)
    for c in range(1, inst.n + 1):
        vs = on.get(c, set())
        best = max((x for v, x in enumerate(rets) if v not in vs), default=0.0)
        for v in vs:
            x = walk([op for op in routes[v] if op // 2 + 1 != c])
            if x > best:
                best = x
        gains[c] = cur - best
    return gains


def _fisher_yates(items, size, rng):
    pool = list(items)
    for i in range(size):
        j = i + int(rng.integers(len(pool) - i))
        pool[i], pool[j] = pool[j], pool[i]
    return pool[:size]


def destroy(inst, ops, lens, operator: str, q: int, rng):
    """ref alns.destroy + insertion.remove_customers on a flat solution.
    Returns (partial ops [2n] -1 padded, partial lens [m], removed sorted)."""
    n = inst.n
    d, _ = inst.arrays()
    routes = _routes(ops, lens)
    q = min(q, n)
    cs = list(range(1, n + 1))
    q_min = min(removal_bounds(n)[0], n)
    if operator in ("shaw", "critical_path"):
        st, z, rets, arrival, times, q0 = O.evaluate_one(inst, ops, lens)
        t_drop = np.zeros(n + 1)
        dveh = np.zeros(n + 1, np.int64)
        pveh = np.zeros(n + 1, np.int64)
        at = 0
        for v, r in enumerate(routes):
            for op in r:
                c = op // 2 + 1
                if op & 1:
                    pveh[c] = v
                else:
                    dveh[c] = v
                    t_drop[c] = times[at]
                at += 1
    if operator == "random":
        picked = _fisher_yates(cs, q, rng)
    elif operator == "worst":
        g = removal_gains(inst, ops, lens)
        ranked = sorted(cs, key=lambda c: (-g[c], c))
        picked = []
        while len(picked) < q:
            idx = int(rng.random() ** WORST_POWER * len(ranked))
            picked.append(ranked.pop(min(idx, len(ranked) - 1)))
    elif operator == "shaw":
        def rel(a, b):
            x = SHAW_W_TRAVEL * d[a][b]
            x += SHAW_W_TIME * abs(t_drop[a] - t_drop[b])
            if dveh[a] != dveh[b]:
                x += SHAW_W_AGENT / 2.0
            if pveh[a] != pveh[b]:
                x += SHAW_W_AGENT / 2.0
            return x
        first = cs[int(rng.integers(n))]
        picked = [first]
        pool = [c for c in cs if c != first]
        while len(picked) < q and pool:
            anchor = picked[int(rng.integers(len(picked)))]
            best = min(pool, key=lambda c: (rel(anchor, c), c))
            pool.remove(best)
            picked.append(best)
    elif operator == "cluster":
        centre = cs[int(rng.integers(n))]
        near = sorted((c for c in cs if c != centre), key=lambda c: (d[centre][c], c))
        picked = [centre] + near[:q - 1]
    elif operator == "route":
        used = [v for v, r in enumerate(routes) if r]
        v = used[int(rng.integers(len(used)))]
        picked = sorted({op // 2 + 1 for op in routes[v]})
        if len(picked) < q_min:
            pool = [c for c in cs if c not in picked]
            while len(picked) < q_min and pool:
                best = min(pool, key=lambda c: (min(d[c][x] for x in picked), c))
                pool.remove(best)
                picked.append(best)
    elif operator == "critical_path":
        v = int(np.argmax(rets))  # Schedule.bottleneck: first maximum
        mine = sorted({op // 2 + 1 for op in routes[v]})
        if len(mine) >= q:
            picked = _fisher_yates(mine, q, rng)
        else:
            picked = list(mine)
            if len(picked) < q_min:
                g = removal_gains(inst, ops, lens)
                rest = sorted((c for c in cs if c not in picked), key=lambda c: (-g[c], c))
                picked.extend(rest[:q_min - len(picked)])
    else:
        raise ValueError(f"unknown destroy operator {operator!r}")
    full, plens, removed = O.remove_customers(inst, ops, lens, picked)
    out = full[:2 * n].copy()
    out[int(plens.sum()):] = -1
    return out, plens, [int(c) for c in removed]
