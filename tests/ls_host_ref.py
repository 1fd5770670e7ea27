"""Host-built local-search neighbourhoods -- TEST INFRASTRUCTURE: the
cross-check of the device-built batch path (paper_2602_23685_b200/
localsearch.py).  The reference's pickup_repositioning /
cross_agent_relocation (alns.py:416-487) restated over numpy op arrays, each
candidate materialised on the host and scored by the device's K2/K1 (so the
test isolates the device neighbourhood builder and the top-10 reduction)."""
from __future__ import annotations

import numpy as np

from paper_2602_23685_b200.schedule import OpKind, Solution, evaluate

_P = OpKind.PICKUP
_NEAR_BOTTLENECK = 0.9
_VERIFY_LIMIT = 10


def _flat(tours, n):
    """Tour lists -> (ops int32 [total], lens int32 [m])."""
    lens = np.array([len(t) for t in tours], np.int32)
    ops = np.fromiter((2 * (c - 1) + (kind is _P) for t in tours for c, kind in t),
                      dtype=np.int32, count=int(lens.sum()))
    return ops, lens


def _score_arrays(instance, cand_ops, cand_lens, mode):
    """One device batch over candidates given as flat op arrays: K2 (mode 2)
    or K1 (mode 0).  Returns numpy (z, status)."""
    from paper_2602_23685_b200.device import makespan_batch
    n = instance.n
    K = len(cand_ops)
    ops = np.full((K, 2 * n), -1, np.int32)
    for j, o in enumerate(cand_ops):
        ops[j, :o.size] = o
    r = makespan_batch(instance, ops, np.stack(cand_lens), mode=mode)
    return r["z"].cpu().numpy(), r["status"].cpu().numpy()


def _apply_best_verified(instance, tours, candidates, z_cur):
    """Stable sort by estimate, exact-score the best _VERIFY_LIMIT (one K1
    batch), keep the strongest strict improvement (alns.py:401-413).
    candidates: [(est, ops, lens)] in generation order."""
    candidates.sort(key=lambda c: c[0])
    top = candidates[:_VERIFY_LIMIT]
    if not top:
        return None
    z, st = _score_arrays(instance, [c[1] for c in top], [c[2] for c in top], 0)
    best = None
    for zi, si, (_, o, l) in zip(z, st, top):
        if si != 0:
            continue
        if zi < z_cur - 1e-9 and (best is None or zi < best[0]):
            best = (float(zi), o, l)
    if best is None:
        return None
    return [list(t) for t in Solution.from_arrays(best[1], best[2]).tours]


def _estimate_filter(instance, cand_ops, cand_lens, z):
    """K2 over all candidates; keep (est, ops, lens) with est < z - 1e-9 in
    generation order (two_pass_estimate errors are skipped)."""
    if not cand_ops:
        return []
    est, st = _score_arrays(instance, cand_ops, cand_lens, 2)
    return [(float(e), o, l) for e, s, o, l in zip(est, st, cand_ops, cand_lens)
            if s == 0 and e < z - 1e-9]


def pickup_repositioning_host(instance, solution: Solution) -> Solution:
    """Host-built neighbourhood variant of pickup_repositioning (candidates as
    numpy op arrays, scored by K2/K1) -- kept as the cross-check of the
    device-built batch path (tests/test_gpu_localsearch.py)."""
    tours = [list(t) for t in solution.tours]
    m = instance.m
    for _ in range(3):
        sched = evaluate(instance, Solution.from_lists(tours))
        z = sched.makespan
        if z <= 0:
            break
        hot = sorted({v for v, r in enumerate(sched.returns) if r >= _NEAR_BOTTLENECK * z})
        ops, lens = _flat(tours, instance.n)
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
        c_ops, c_lens = [], []
        for v in hot:
            for i in range(int(lens[v])):
                op = int(ops[starts[v] + i])
                if not op & 1:
                    continue
                base = np.delete(ops, starts[v] + i)
                blens = lens.copy()
                blens[v] -= 1
                bstarts = np.concatenate([[0], np.cumsum(blens)[:-1]])
                for w in range(m):
                    for g in range(int(blens[w]) + 1):
                        if w == v and g == i:
                            continue
                        cl = blens.copy()
                        cl[w] += 1
                        c_ops.append(np.insert(base, bstarts[w] + g, op))
                        c_lens.append(cl)
        new_tours = _apply_best_verified(instance, tours, _estimate_filter(instance, c_ops, c_lens, z), z)
        if new_tours is None:
            break
        tours = new_tours
    return Solution.from_lists(tours)


def cross_agent_relocation_host(instance, solution: Solution) -> Solution:
    """Host-built neighbourhood variant of cross_agent_relocation (cross-check)."""
    if instance.m == 1:
        return solution
    tours = [list(t) for t in solution.tours]
    m = instance.m
    for _ in range(3):
        sched = evaluate(instance, Solution.from_lists(tours))
        z = sched.makespan
        b = sched.bottleneck()
        ops, lens = _flat(tours, instance.n)
        c_ops, c_lens = [], []
        for c in sorted({c for c, _ in tours[b]}):
            keep = (ops >> 1) + 1 != c
            stripped = ops[keep]
            slens = lens.copy()
            at = 0
            for v in range(m):
                slens[v] = int(keep[at:at + lens[v]].sum())
                at += int(lens[v])
            sstarts = np.concatenate([[0], np.cumsum(slens)[:-1]])
            d_op, p_op = 2 * (c - 1), 2 * (c - 1) + 1
            for w in range(m):
                if w == b:
                    continue
                L = int(slens[w])
                cl = slens.copy()
                cl[w] += 2
                for gd in range(L + 1):
                    with_d = np.insert(stripped, sstarts[w] + gd, d_op)
                    for gp in range(gd + 1, L + 2):
                        c_ops.append(np.insert(with_d, sstarts[w] + gp, p_op))
                        c_lens.append(cl)
        new_tours = _apply_best_verified(instance, tours, _estimate_filter(instance, c_ops, c_lens, z), z)
        if new_tours is None:
            break
        tours = new_tours
    return Solution.from_lists(tours)


# The entry lists of one local-search pass built on the host from numpy arrays
# (the reference's generation order, alns.py:416-487) -- the checker of the
# device builder vrp_ls_entries (localsearch.entries).
NEAR_BOTTLENECK = _NEAR_BOTTLENECK


def pickup_entries(ops, lens, z, returns, active):
    m = lens.shape[1]
    ent, alive = [], []
    for w in active:
        if z[w] <= 0:
            continue
        alive.append(w)
        off = np.concatenate([[0], np.cumsum(lens[w])[:-1]])
        for v in range(m):
            if not returns[w, v] >= NEAR_BOTTLENECK * z[w]:
                continue
            seg = ops[w, off[v]:off[v] + lens[w, v]]
            for i in np.flatnonzero(seg & 1):
                ent.append((w, v, int(i), int(off[v] + i), 0))
    return ent, alive


def cross_entries(ops, lens, z, returns, active):
    m = lens.shape[1]
    ent, cnt = [], []
    for w in active:
        b = int(np.argmax(returns[w]))  # Schedule.bottleneck: first max
        off = np.concatenate([[0], np.cumsum(lens[w])[:-1]])
        total = int(lens[w].sum())
        flat = ops[w, :total]
        cust = (flat >> 1) + 1
        route = np.repeat(np.arange(m), lens[w])
        for c in sorted(set(cust[off[b]:off[b] + lens[w, b]].tolist())):
            pos = np.flatnonzero(cust == c)
            f1, f2 = int(pos[0]), int(pos[1])
            for u in range(m):
                if u == b:
                    continue
                L = int(lens[w, u]) - int((route[pos] == u).sum())
                ent.append((w, c, u, f1, f2))
                cnt.append((L + 1) * (L + 2) // 2)
    return ent, np.asarray(cnt, np.int64)
