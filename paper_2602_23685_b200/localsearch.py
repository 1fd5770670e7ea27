"""Batched local search on the device: the reference's
``pickup_repositioning`` and ``cross_agent_relocation`` (alns.py:401-487) for
many solutions at once.

Each improvement pass of every solution is:
  1. K1 ``evaluate`` of the current solutions (returns -> hot vehicles / the
     bottleneck), one launch for all of them;
  2. the neighbourhood entries built on the device from those returns
     (``vrp_ls_entries``: a count launch, the host scans W counts, a fill
     launch), then the candidates, numbered in the reference's generation
     order, built chunk by chunk (``vrp_ls_build``) and estimated by K2
     ``two_pass_estimate`` -- solutions never leave the device;
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


def _search(instance, kind, ops_t, lens_t, ent_t, start_t, ccount, coff, z):
    """Steps 2-4 for the solutions that have entries (device tables ent_t /
    start_t, per-solution candidate counts / offsets on the host).  Returns
    {worker: (z_exact, ops row, lens row)} for the workers that improved."""
    dev = ops_t.device
    n = instance.n
    W = ops_t.shape[0]
    total = int(ccount.sum())
    zthr = torch.from_numpy(np.asarray(z, np.float64) - 1e-9).to(dev)
    # each solution's candidates are one contiguous range (entries are grouped by solution)
    wid = np.flatnonzero(ccount > 0)
    wb = coff[wid]
    we = wb + ccount[wid]
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


def entries(instance, kind, ops_t, lens_t, z, returns, active):
    """The pass's neighbourhood entries, built on the device (vrp_ls_entries).
    z [W] / returns [W, m] host arrays, active: worker indices.  Returns
    (entries int32 [E, 5] device, entry_start int64 [E] device, per-solution
    candidate counts and offsets (numpy int64 [W]))."""
    dev = ops_t.device
    di = DV.device_instance(instance)
    W = ops_t.shape[0]
    act = np.zeros(W, np.uint8)
    act[np.asarray(list(active), np.int64)] = 1
    z_t = torch.from_numpy(np.ascontiguousarray(z, np.float64)).to(dev)
    r_t = torch.from_numpy(np.ascontiguousarray(returns, np.float64)).to(dev)
    a_t = torch.from_numpy(act).to(dev)
    ec = torch.empty(W, dtype=torch.int32, device=dev)
    cc = torch.empty(W, dtype=torch.int64, device=dev)
    L, h, s = N.lib(), di.handle, N.stream_handle()
    N.check(L.vrp_ls_entries(h, kind, N.ptr(ops_t), N.ptr(lens_t), N.ptr(z_t), N.ptr(r_t), N.ptr(a_t), W,
                             None, None, N.ptr(ec), N.ptr(cc), None, None, s), "vrp_ls_entries")
    ecount, ccount = ec.cpu().numpy().astype(np.int64), cc.cpu().numpy()
    eoff = np.zeros(W, np.int64)
    coff = np.zeros(W, np.int64)
    np.cumsum(ecount[:-1], out=eoff[1:])
    np.cumsum(ccount[:-1], out=coff[1:])
    E = int(ecount.sum())
    ent_t = torch.empty((max(E, 1), 5), dtype=torch.int32, device=dev)
    start_t = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
    if E:
        eo, co = torch.from_numpy(eoff).to(dev), torch.from_numpy(coff).to(dev)
        N.check(L.vrp_ls_entries(h, kind, N.ptr(ops_t), N.ptr(lens_t), N.ptr(z_t), N.ptr(r_t), N.ptr(a_t), W,
                                 N.ptr(eo), N.ptr(co), None, None, N.ptr(ent_t), N.ptr(start_t), s),
                "vrp_ls_entries")
    return ent_t[:E], start_t[:E], ccount, coff


def _run(instance, kind, ops, lens):
    """ops [W, 2n] int32, lens [W, m] int32 (numpy or device tensors) ->
    (ops, lens) device tensors after the passes, z_exact numpy [W]."""
    dev = torch.device("cuda", torch.cuda.current_device())
    ops_t = torch.as_tensor(ops, dtype=torch.int32).to(dev).contiguous().clone()
    lens_t = torch.as_tensor(lens, dtype=torch.int32).to(dev).contiguous().clone()
    W, m = ops_t.shape[0], instance.m
    z, returns = _evaluate(instance, ops_t, lens_t)
    z_out = z.copy()
    if kind == 1 and m == 1:
        return ops_t, lens_t, z_out
    active = list(range(W))
    for _ in range(PASSES):
        if not active:
            break
        ent_t, start_t, ccount, coff = entries(instance, kind, ops_t, lens_t, z, returns, active)
        if not ent_t.shape[0]:
            break
        res = _search(instance, kind, ops_t, lens_t, ent_t, start_t, ccount, coff, z)
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
