"""Device-built local search (localsearch.py, vrp_ls_build + K2/K1) against
the reference's goldens and the host-built neighbourhoods, batched."""
import numpy as np
import pytest
import torch

import inputs as I
from conftest import config_instance
from oracle import oracle as O
import ls_host_ref as H
from paper_2602_23685_b200 import alns as A
from paper_2602_23685_b200 import localsearch as LS
from paper_2602_23685_b200.schedule import Solution, exact_makespan

pytestmark = pytest.mark.gpu
CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


@pytest.mark.parametrize("key", ["gr17", "eil51", "kroA100"])
def test_batched_local_search_matches_reference(key, golden):
    inst = config_instance(key)
    ops = golden[f"{key}/dec_ops"][:3]
    lens = golden[f"{key}/dec_lens"][:3]
    for tag, fn in (("pr", LS.pickup_repositioning_batch), ("ca", LS.cross_agent_relocation_batch)):
        o, l, z = fn(inst, ops, lens)
        for j in range(3):
            np.testing.assert_array_equal(l[j].cpu().numpy(), golden[f"ls/{key}/{tag}/{j}/lens"], err_msg=f"{tag} {j}")
            np.testing.assert_array_equal(o[j].cpu().numpy(), golden[f"ls/{key}/{tag}/{j}/ops"], err_msg=f"{tag} {j}")
            assert z[j] == exact_makespan(inst, Solution.from_arrays(o[j].cpu().numpy(), l[j].cpu().numpy()))


@pytest.mark.parametrize("key,count", [("gr17", 24), ("eil51", 16), ("kroA100", 8), ("a280", 3)])
def test_batched_local_search_vs_host_neighbourhoods(key, count):
    """Fresh decoded solutions (several per batch, some already improved by a
    first call) against the host-built variant, both LS kinds."""
    inst = config_instance(key)
    genes = I.chromosomes(inst.n, count, (83, CID[key]))
    dec = O.decode_batch(inst, genes)
    ops, lens = dec["ops"], dec["lens"]
    for kind, fn, host in ((0, LS.pickup_repositioning_batch, H.pickup_repositioning_host),
                           (1, LS.cross_agent_relocation_batch, H.cross_agent_relocation_host)):
        o, l, z = fn(inst, ops, lens)
        o, l = o.cpu().numpy(), l.cpu().numpy()
        for j in range(count):
            ref = host(inst, Solution.from_arrays(ops[j], lens[j]))
            ro, rl = ref.to_arrays(inst.n)
            np.testing.assert_array_equal(l[j], rl, err_msg=f"{kind} {j}")
            np.testing.assert_array_equal(o[j], ro[:2 * inst.n], err_msg=f"{kind} {j}")
            assert z[j] == exact_makespan(inst, ref)


def test_builder_covers_whole_neighbourhood():
    """Every candidate of a small cross neighbourhood is a valid permutation
    of the ops with c's pair on w in (gd < gp) order, each exactly once."""
    inst = config_instance("gr17")
    dec = O.decode_batch(inst, I.chromosomes(inst.n, 1, (5, 5)))
    ops = torch.from_numpy(dec["ops"]).cuda()
    lens = torch.from_numpy(dec["lens"]).cuda()
    o, l = dec["ops"][0], dec["lens"][0]
    c = int(o[0] >> 1) + 1
    pos = np.flatnonzero((o >> 1) + 1 == c)
    ent = []
    cnt = []
    for u in range(inst.m):
        L = int(l[u]) - int(sum(1 for p in pos if sum(l[:u]) <= p < sum(l[:u + 1])))
        ent.append((0, c, u, int(pos[0]), int(pos[1])))
        cnt.append((L + 1) * (L + 2) // 2)
    starts = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    total = int(sum(cnt))
    b_ops, b_lens = LS._build(inst, 1, ops, lens, torch.tensor(ent, dtype=torch.int32).cuda(),
                              torch.from_numpy(starts).cuda(), 0, total, op_dtype=torch.int32)
    b_ops, b_lens = b_ops.cpu().numpy(), b_lens.cpu().numpy()
    seen = set()
    for j in range(total):
        assert sorted(b_ops[j].tolist()) == sorted(o.tolist())
        seen.add(tuple(b_ops[j].tolist()) + tuple(b_lens[j].tolist()))
    assert len(seen) == total


def test_ls_topk_kernel_vs_numpy():
    """vrp_ls_topk: per solution, the K smallest (estimate, generation index)
    survivors (status 0, estimate < threshold) over several chunks -- the
    reference's stable sort + [:_VERIFY_LIMIT] -- against numpy."""
    from paper_2602_23685_b200 import _native as N
    from paper_2602_23685_b200.localsearch import _segments
    g = np.random.default_rng(5)
    W, K = 7, 10
    sizes = np.array([0, 5, 3000, 1, 9000, 17, 4200])  # candidates per solution (ranges ascending)
    wb = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    we = wb + sizes
    total = int(sizes.sum())
    z = np.round(g.random(total) * 50) / 4  # many ties
    st = (g.random(total) < 0.1).astype(np.int32)
    thr = g.random(W) * 12
    wid = np.flatnonzero(sizes > 0)
    dev = torch.device("cuda")
    top_z = torch.empty((W, K), dtype=torch.float64, device=dev)
    top_i = torch.empty((W, K), dtype=torch.int64, device=dev)
    top_n = torch.from_numpy(np.zeros(W, np.int32)).to(dev)
    zthr = torch.from_numpy(thr).to(dev)
    chunk = 2500
    for first in range(0, total, chunk):
        cnt = min(chunk, total - first)
        zz = torch.from_numpy(z[first:first + cnt].copy()).to(dev)
        ss = torch.from_numpy(st[first:first + cnt].copy()).to(dev)
        tabs = [torch.from_numpy(x).to(dev) for x in _segments(wid, wb[wid], we[wid], first, cnt)]
        seg_w, seg_b, seg_e, ws, wf, wc = tabs
        N.check(N.lib().vrp_ls_topk(N.ptr(zz), N.ptr(ss), first, N.ptr(zthr), N.ptr(seg_w), N.ptr(seg_b),
                                    N.ptr(seg_e), seg_w.numel(), N.ptr(ws), N.ptr(wf), N.ptr(wc), ws.numel(), K,
                                    N.ptr(top_z), N.ptr(top_i), N.ptr(top_n), N.stream_handle()), "vrp_ls_topk")
    tn, tz, ti = top_n.cpu().numpy(), top_z.cpu().numpy(), top_i.cpu().numpy()
    for w in range(W):
        idx = np.arange(wb[w], we[w])
        ok = idx[(st[idx] == 0) & (z[idx] < thr[w])]
        order = ok[np.lexsort((ok, z[ok]))][:K]  # stable by estimate
        assert tn[w] == order.size, w
        np.testing.assert_array_equal(ti[w, :tn[w]], order)
        np.testing.assert_array_equal(tz[w, :tn[w]], z[order])


@pytest.mark.gpu
@pytest.mark.parametrize("key,count", [("gr17", 12), ("eil51", 9), ("a280", 5), ("dsj1000", 4)])
def test_ls_entries_kernel_vs_host(key, count):
    """vrp_ls_entries (both kinds) equals the host entry builders: same
    entries in the same order, same candidate starts, on a subset of active
    solutions, with one vehicle's return set exactly to 0.9 z (kept: >=)."""
    inst = config_instance(key)
    dec = O.decode_batch(inst, I.chromosomes(inst.n, count, (84, CID.get(key, 9))))
    ops, lens = dec["ops"].astype(np.int32), dec["lens"].astype(np.int32)
    ops_t, lens_t = torch.from_numpy(ops).cuda(), torch.from_numpy(lens).cuda()
    z, returns = LS._evaluate(inst, ops_t, lens_t)
    returns = returns.copy()
    v = int(np.argmin(returns[0]))
    returns[0, v] = 0.9 * z[0]
    active = [w for w in range(count) if w % 3 != 1]
    for kind in (0, 1):
        ent_t, start_t, ccount, coff = LS.entries(inst, kind, ops_t, lens_t, z, returns, active)
        if kind == 0:
            ent, _ = H.pickup_entries(ops, lens, z, returns, active)
            cnt = np.full(len(ent), 2 * inst.n + inst.m - 2, np.int64)
        else:
            ent, cnt = H.cross_entries(ops, lens, z, returns, active)
        ent = np.asarray(ent, np.int32).reshape(-1, 5)
        starts = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
        np.testing.assert_array_equal(ent_t.cpu().numpy(), ent, err_msg=f"kind {kind}")
        np.testing.assert_array_equal(start_t.cpu().numpy(), starts, err_msg=f"kind {kind}")
        per = np.zeros(count, np.int64)
        np.add.at(per, ent[:, 0], cnt)
        np.testing.assert_array_equal(ccount, per)
