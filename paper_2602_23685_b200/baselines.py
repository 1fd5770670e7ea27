"""Heuristic polish on the device -- drop-in for the reference's
``baselines.two_opt_improve`` (``/root/reference/pkg/src/vrp_rpd/baselines.py:372-455``,
SURVEY §8(f) row 3).

The reference scans three neighbourhoods in a fixed order -- intra-route
2-opt reversal, single-operation relocation, pairwise swap -- re-scoring every
candidate with ``evaluate`` and taking the FIRST strict improvement
(< best - 1e-9), restarting from 2-opt after each one, until a fixed point or
the move budget (default 50n evaluated candidates) runs out.

Here each scan is evaluated chunk by chunk: ``vrp_ls_build`` materialises the
next candidates of the current neighbourhood in the reference's order
(kinds 2 / 0 / 3), K1 scores them with ``evaluate`` semantics, and the first
improving index in the chunk is exactly the reference's next accepted move
(everything before it was non-improving).  The budget is charged as the
reference charges it: the candidates up to and including the accepted one,
or the whole chunk when none improves; chunks never exceed the remaining
budget.  Candidates evaluated past the accepted one are speculation the
reference never sees, so the result is bit-identical."""
from __future__ import annotations

import time

import numpy as np
import torch

from . import _native as N
from . import device as DV
from .localsearch import _build
from .schedule import Solution, evaluate

CHUNK = 1 << 15


def _phase_entries(kind, lens, n):
    """Entries + candidate counts of one neighbourhood (zero-count entries
    dropped so that entry_start stays strictly increasing)."""
    m = lens.size
    L = np.asarray(lens, np.int64)
    if kind == 2:  # 2-opt: routes in order
        vs = np.flatnonzero(L >= 2)
        ent = np.zeros((vs.size, 5), np.int32)
        ent[:, 1] = vs
        cnt = L[vs] * (L[vs] - 1) // 2
    elif kind == 0:  # relocation: every op in route order
        total = int(L.sum())
        off = np.cumsum(L) - L
        v = np.repeat(np.arange(m), L)
        ent = np.zeros((total, 5), np.int32)
        ent[:, 1] = v
        ent[:, 3] = np.arange(total)
        ent[:, 2] = ent[:, 3] - off[v]
        cnt = np.full(total, 2 * n + m - 2, np.int64)
    else:  # swap: one entry, all flat pairs
        ent = np.zeros((1, 5), np.int32)
        cnt = np.array([2 * n * (2 * n - 1) // 2], np.int64)
    return ent, cnt


def two_opt_improve(instance, solution: Solution, move_budget: int | None = None,
                    chunk: int = CHUNK, deadline: float | None = None, resume: bool = False,
                    max_chunk: int = 1 << 20) -> Solution:
    """First-improvement 2-opt / relocate / swap polish (baselines.py:372-455).

    The chunk doubles (up to ``max_chunk``) after every chunk without an
    improvement and falls back to ``chunk`` after one -- fewer launches on
    long fruitless scans, same result (any chunking takes the same first
    improvement).  Two extensions beyond the reference, off by default:
    ``deadline`` (time.perf_counter() value) stops between chunks, and
    ``resume`` continues the scan after an improvement from where it was
    (cycling through the three neighbourhoods, stopping after one full
    fruitless cycle) instead of restarting at 2-opt -- a different, faster
    local search, used by the time-budgeted pipeline."""
    n = instance.n
    budget = move_budget if move_budget is not None else 50 * n
    dev = torch.device("cuda", torch.cuda.current_device())
    op_dtype = torch.int16 if 2 * n <= 32767 else torch.int32
    o, l = solution.to_arrays(n)
    ops_t = torch.from_numpy(np.ascontiguousarray(o[None, :2 * n])).to(dev)
    lens_t = torch.from_numpy(np.ascontiguousarray(l[None])).to(dev)
    best = evaluate(instance, solution).makespan
    kinds = (2, 0, 3)
    phase, pos = 0, 0          # resume point
    fruitless = 0              # resume: candidates scanned since the last improvement
    step = chunk
    improved = True
    while improved and budget > 0:
        improved = False
        lens = lens_t[0].cpu().numpy()
        tables = [_phase_entries(k, lens, n) for k in kinds]
        grand = sum(int(c.sum()) for _, c in tables)
        if not resume:
            phase, pos = 0, 0
        for turn in range(3 if not resume else 4):
            ph = (phase + turn) % 3 if resume else turn
            kind = kinds[ph]
            ent, cnt = tables[ph]
            total = int(cnt.sum())
            if total == 0:
                continue
            starts = np.zeros(len(cnt), np.int64)
            np.cumsum(cnt[:-1], out=starts[1:])
            ent_t = torch.from_numpy(ent).to(dev)
            start_t = torch.from_numpy(starts).to(dev)
            p0 = pos if (resume and turn == 0) else 0
            p = min(p0, total)
            while p < total and budget > 0:
                if deadline is not None and time.perf_counter() >= deadline:
                    budget = 0
                    break
                if resume and fruitless >= grand:
                    budget = 0  # a whole cycle without improvement: local optimum
                    break
                k = min(step, total - p, budget)
                c_ops, c_lens = _build(instance, kind, ops_t, lens_t, ent_t, start_t, p, k,
                                       op_dtype=op_dtype)
                # candidates are permutations of a valid solution, so evaluate()'s
                # structural check never fires and K1's exact mode gives the same
                # status and makespan (CAPACITY before DEADLOCK in both)
                r = DV.makespan_batch(instance, c_ops, c_lens, mode=N.MODE_EXACT)
                ok = (r["status"] == 0) & (r["z"] < best - 1e-9)
                hit = torch.nonzero(ok)
                if hit.numel():
                    j = int(hit[0, 0])
                    budget -= j + 1
                    best = float(r["z"][j])
                    ops_t = c_ops[j:j + 1].to(torch.int32)
                    lens_t = c_lens[j:j + 1].clone()
                    improved = True
                    phase, pos, fruitless, step = ph, p + j + 1, 0, chunk
                    break
                budget -= k
                fruitless += k
                p += k
                step = min(2 * step, max_chunk)
            if improved or budget <= 0:
                break
    return Solution.from_arrays(ops_t[0].cpu().numpy(), lens_t[0].cpu().numpy())
