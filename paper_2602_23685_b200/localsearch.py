"""Batched local search on the device: the reference's
``pickup_repositioning`` and ``cross_agent_relocation`` (alns.py:401-487) for
many solutions at once.

Each improvement pass of every solution is:
  1. K1 ``evaluate`` of the current solutions (returns -> hot vehicles / the
     bottleneck), one launch for all of them;
  2. the neighbourhood, numbered in the reference's generation order, built
     chunk by chunk on the device (``vrp_ls_build``) and estimated by K2
     ``two_pass_estimate`` -- nothing is materialised on the host;
  3. survivors (status 0, estimate < z - 1e-9) reduced on the device to each
     solution's ten best by (estimate, generation index) -- the reference's
     stable sort + ``[:_VERIFY_LIMIT]`` -- by ``vrp_ls_topk`` (per-segment
     block top-10, then a per-solution merge with the running list);
  4. those ten re-built and scored by K1 ``exact_makespan``; the first strictly
     best improvement (< z - 1e-9) replaces the solution (alns.py:401-413).
A solution leaves the loop when a pass finds nothing, exactly like the
reference's ``break``.  Results are bit-identical to the reference
(tests/test_gpu_localsearch.py)."""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from . import device as DV

NEAR_BOTTLENECK = 0.9   # alns.py:_NEAR_BOTTLENECK
VERIFY_LIMIT = 10       # alns.py:_VERIFY_LIMIT
PASSES = 3
CHUNK_BYTES = 1 << 30   # candidate ops per K2 chunk


def _build(instance, kind, ops_t, lens_t, ent_t, start_t, first, count, index_list=None, op_dtype=torch.int16):
    di = DV.device_instance(instance)
    n, m = instance.n, instance.m
    out = torch.empty((count, 2 * n), dtype=op_dtype, device=ops_t.device)
    olen = torch.empty((count, m), dtype=torch.int32, device=ops_t.device)
    N.check(N.lib().vrp_ls_build(di.handle, kind, N.ptr(ops_t), N.ptr(lens_t), N.ptr(ent_t),
                                 N.ptr(start_t), ent_t.shape[0], N.ptr(index_list), int(first), int(count),
                                 N.ptr(out), out.element_size(), N.ptr(olen), N.stream_handle()),
            "vrp_ls_build")
    return out, olen


SEG = 2048  # candidates per top-K segment (csrc/ls.cu LS_SEG)


def _segments(wid, wb, we, first, cnt):
    """Segments of <= SEG candidates of one solution each covering the chunk
    [first, first + cnt) (solutions' candidate ranges [wb, we) are disjoint
    and ascending).  Returns the vrp_ls_topk tables (numpy)."""
    lo = np.maximum(wb, first)
    hi = np.minimum(we, first + cnt)
    live = np.flatnonzero(hi > lo)
    lo, hi, wid = lo[live], hi[live], wid[live]
    nseg = (hi - lo + SEG - 1) // SEG
    seg_w = np.repeat(wid, nseg).astype(np.int32)
    k = np.arange(int(nseg.sum())) - np.repeat(np.cumsum(nseg) - nseg, nseg)
    seg_b = np.repeat(lo, nseg) + SEG * k
    seg_e = np.minimum(seg_b + SEG, np.repeat(hi, nseg))
    wfirst = (np.cumsum(nseg) - nseg).astype(np.int32)
    return seg_w, seg_b.astype(np.int64), seg_e.astype(np.int64), wid.astype(np.int32), wfirst, nseg.astype(np.int32)


def _search(instance, kind, ops_t, lens_t, entries, counts, z):
    """Steps 2-4 for every worker that has entries.  Returns
    {worker: (z_exact, ops row, lens row)} for the workers that improved."""
    dev = ops_t.device
    n = instance.n
    W = ops_t.shape[0]
    starts = np.zeros(len(counts), np.int64)
    np.cumsum(counts[:-1], out=starts[1:])
    total = int(counts.sum())
    ent_t = torch.from_numpy(np.ascontiguousarray(entries, np.int32)).to(dev)
    start_t = torch.from_numpy(starts).to(dev)
    zthr = torch.from_numpy(np.asarray(z, np.float64) - 1e-9).to(dev)
    # each solution's candidates are one contiguous range (entries are grouped by solution)
    ew = np.asarray(entries, np.int64)[:, 0]
    wid, pos = np.unique(ew, return_index=True)
    last = np.r_[pos[1:], ew.size] - 1
    wb, we = starts[pos], starts[last] + counts[last]
    # running lists: only the first top_n entries are ever read (no fill kernels)
    top_z = torch.empty((W, VERIFY_LIMIT), dtype=torch.float64, device=dev)
    top_i = torch.empty((W, VERIFY_LIMIT), dtype=torch.int64, device=dev)
    top_n = torch.from_numpy(np.zeros(W, np.int32)).to(dev)
    chunk = max(1, CHUNK_BYTES // (4 * n))
    for first in range(0, total, chunk):
        cnt = min(chunk, total - first)
        c_ops, c_lens = _build(instance, kind, ops_t, lens_t, ent_t, start_t, first, cnt)
        r = DV.makespan_batch(instance, c_ops, c_lens, mode=N.MODE_TWO_PASS)
        seg_w, seg_b, seg_e, ws, wf, wc = (torch.from_numpy(x).to(dev) for x in _segments(wid, wb, we, first, cnt))
        N.check(N.lib().vrp_ls_topk(N.ptr(r["z"]), N.ptr(r["status"]), first, N.ptr(zthr), N.ptr(seg_w),
                                    N.ptr(seg_b), N.ptr(seg_e), seg_w.numel(), N.ptr(ws), N.ptr(wf), N.ptr(wc),
                                    ws.numel(), VERIFY_LIMIT, N.ptr(top_z), N.ptr(top_i), N.ptr(top_n),
                                    N.stream_handle()), "vrp_ls_topk")
    tn = top_n.cpu().numpy()
    if not tn.any():
        return {}
    ti = top_i.cpu().numpy()
    sel_w = np.repeat(np.arange(W), tn)  # (worker, estimate, index) order
    sel_i = np.concatenate([ti[w, :tn[w]] for w in range(W) if tn[w]])
    v_ops, v_lens = _build(instance, kind, ops_t, lens_t, ent_t, start_t, 0, sel_i.size,
                           index_list=torch.from_numpy(sel_i).to(dev), op_dtype=torch.int32)
    r = DV.makespan_batch(instance, v_ops, v_lens, mode=N.MODE_EXACT)
    zs, st = r["z"].cpu().numpy(), r["status"].cpu().numpy()
    best = {}
    for j in range(sel_w.size):
        w = int(sel_w[j])
        if st[j] != 0 or not zs[j] < z[w] - 1e-9:
            continue
        if w not in best or zs[j] < best[w][0]:
            best[w] = (float(zs[j]), j)
    return {w: (zb, v_ops[j], v_lens[j]) for w, (zb, j) in best.items()}


def _evaluate(instance, ops_t, lens_t):
    r = DV.makespan_batch(instance, ops_t, lens_t, mode=N.MODE_EVALUATE, want_returns=True)
    st = r["status"].cpu().numpy()
    if (st != 0).any():
        raise ValueError("local search needs valid solutions")
    return r["z"].cpu().numpy(), r["returns"].cpu().numpy()


def _pickup_entries(ops, lens, z, returns, active):
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


def _cross_entries(ops, lens, z, returns, active):
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


def _run(instance, kind, ops, lens):
    """ops [W, 2n] int32, lens [W, m] int32 (numpy or device tensors) ->
    (ops, lens) device tensors after the passes, z_exact numpy [W]."""
    dev = torch.device("cuda", torch.cuda.current_device())
    ops_t = torch.as_tensor(ops, dtype=torch.int32).to(dev).contiguous().clone()
    lens_t = torch.as_tensor(lens, dtype=torch.int32).to(dev).contiguous().clone()
    W, m, n = ops_t.shape[0], instance.m, instance.n
    z, returns = _evaluate(instance, ops_t, lens_t)
    z_out = z.copy()
    if kind == 1 and m == 1:
        return ops_t, lens_t, z_out
    active = list(range(W))
    for _ in range(PASSES):
        if not active:
            break
        ops_np, lens_np = ops_t.cpu().numpy(), lens_t.cpu().numpy()
        if kind == 0:
            ent, active = _pickup_entries(ops_np, lens_np, z, returns, active)
            counts = np.full(len(ent), 2 * n + m - 2, np.int64)
        else:
            ent, counts = _cross_entries(ops_np, lens_np, z, returns, active)
        if not ent:
            break
        res = _search(instance, kind, ops_t, lens_t, np.asarray(ent, np.int32), counts, z)
        active = sorted(res)
        for w, (zb, o, l) in res.items():
            ops_t[w] = o
            lens_t[w] = l
            z_out[w] = zb
        if active:
            z2, r2 = _evaluate(instance, ops_t, lens_t)
            z[active], returns[active] = z2[active], r2[active]
    return ops_t, lens_t, z_out


def pickup_repositioning_batch(instance, ops, lens):
    """alns.pickup_repositioning (alns.py:416-450) for every row; returns
    (ops, lens) device tensors and the exact makespans (numpy)."""
    return _run(instance, 0, ops, lens)


def cross_agent_relocation_batch(instance, ops, lens):
    """alns.cross_agent_relocation (alns.py:453-487) for every row."""
    return _run(instance, 1, ops, lens)
