"""Edge-case parity sweep: many tiny random instances (n down to 1, m and k
down to 1, more vehicles than customers, empty routes, a route holding every
op, symmetric and asymmetric integral distances, non-integral distances)
through K1/K2 (all three modes), K3 decode, K5 repair and K6 destroy --
against the CPU oracle, or the host destroy where the oracle has none."""
import numpy as np
import pytest
import torch

import inputs as I
from oracle import destroy_oracle as DO
from oracle import oracle as O
from paper_2602_23685_b200 import alns as A
from paper_2602_23685_b200 import device as DV
from paper_2602_23685_b200 import insertion as INS
from paper_2602_23685_b200 import rng as R
from paper_2602_23685_b200.instance import Instance
from paper_2602_23685_b200.schedule import Solution

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1, 1), (1, 3, 1), (2, 1, 1), (2, 2, 1), (3, 5, 2), (4, 1, 3), (5, 2, 1), (6, 3, 2),
          (8, 8, 1), (9, 2, 4), (12, 4, 2), (17, 3, 5), (20, 8, 5), (12, 7, 6)]  # last two: m*k > 32 (narrow K1)


def _instance(n, m, k, seed, kind):
    g = np.random.default_rng(seed)
    xy = g.integers(0, 60, size=(n + 1, 2))
    d = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1))
    if kind == "int":
        d = np.rint(d)
    elif kind == "asym":
        d = np.rint(d + g.integers(0, 9, size=d.shape))
        np.fill_diagonal(d, 0)
    else:  # fractional
        d = d + g.random(d.shape) / 3
        np.fill_diagonal(d, 0)
    p = g.integers(1, 40, size=n + 1).astype(float)
    p[0] = 0
    if kind == "frac":
        p = p + g.random(n + 1) / 7
        p[0] = 0
    return Instance.from_arrays(d, p, m, k, label=f"edge-{n}-{m}-{k}-{kind}")


def _cases():
    for i, (n, m, k) in enumerate(SHAPES):
        for kind in ("int", "asym", "frac"):
            yield i, n, m, k, kind


@pytest.mark.parametrize("i,n,m,k,kind", list(_cases()))
def test_tiny_instances_all_kernels(i, n, m, k, kind):
    inst = _instance(n, m, k, 1000 + i, kind)
    # K3 decode (relaxed and strict) vs oracle
    genes = I.chromosomes(n, 64, (900, i))
    for relax in (True, False):
        r = DV.decode_batch(inst, torch.from_numpy(genes).cuda(), relax=relax)
        ref = O.decode_batch(inst, genes, relax=relax)
        np.testing.assert_array_equal(r["ops"].cpu().numpy(), ref["ops"])
        np.testing.assert_array_equal(r["lens"].cpu().numpy(), ref["lens"])
        np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
    dec = O.decode_batch(inst, genes)
    # K1/K2: decoded, random (capacity / deadlock heavy), every op on one vehicle,
    # and swap-perturbed candidates
    rops, rlens = I.random_candidates(n, m, 64, (901, i))
    one = np.tile(dec["ops"][:1], (4, 1))
    one_l = np.zeros((4, m), np.int32)
    one_l[np.arange(4), np.arange(4) % m] = 2 * n
    ops = np.concatenate([dec["ops"], rops, one, I.swap_perturb(dec["ops"], dec["lens"], (902, i))])
    lens = np.concatenate([dec["lens"], rlens, one_l, dec["lens"]])
    for mode, name in ((0, "exact"), (1, "evaluate"), (2, "two_pass")):
        for dt in (np.int16, np.int32):
            s = DV.makespan_batch(inst, torch.from_numpy(ops.astype(dt)).cuda(), torch.from_numpy(lens).cuda(),
                                  mode=mode, want_returns=True)
            z, st = O.makespan_batch(inst, ops, lens, mode=name)
            np.testing.assert_array_equal(s["status"].cpu().numpy(), st, err_msg=name)
            np.testing.assert_array_equal(s["z"].cpu().numpy(), z, err_msg=name)
    # K5 repair of random removals, all regret kinds, with and without rng
    parts, plens, rem, rks = [], [], [], []
    for j in range(16):
        q = 1 + j % max(1, n)
        pick = I.philox(903, i, j).choice(np.arange(1, n + 1), size=min(q, n), replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][j], dec["lens"][j], pick)
        parts.append(o[:2 * n]); plens.append(l); rem.append(r)
        rks.append((0, 2, 3, m)[j % 4])
    parts, plens = np.stack(parts), np.stack(plens)
    for use in (True, False):
        gens = [I.philox(904, i, j) for j in range(16)] if use else None
        o, l, st = INS.reinsert_batch(inst, parts, plens, rem, rks, gens)
        for j in range(16):
            g = I.philox(904, i, j) if use else None
            rst, ro, rl = O.reinsert_all(inst, parts[j], plens[j], rem[j], rks[j], g)
            assert st[j] == rst, (j, use)
            if rst == 0:
                np.testing.assert_array_equal(o[j], ro)
                np.testing.assert_array_equal(l[j], rl)
            if use:
                assert np.array_equal(R.state_bytes(g), R.state_bytes(gens[j]))
    # K6 destroy vs the host operators (every operator, q across its range)
    sols = [Solution.from_arrays(dec["ops"][j], dec["lens"][j]) for j in range(12)]
    names = [A.DESTROY_OPERATORS[j % 6] for j in range(12)]
    qs = [1 + (j * 3) % n for j in range(12)]
    states = torch.from_numpy(np.stack([R.state_bytes(I.philox(905, i, j)) for j in range(12)])).cuda()
    r = DV.destroy_batch(inst, torch.from_numpy(dec["ops"][:12]).cuda(), torch.from_numpy(dec["lens"][:12]).cuda(),
                         torch.tensor([DV.DESTROY_CODES[x] for x in names], dtype=torch.int32).cuda(),
                         torch.tensor(qs, dtype=torch.int32).cuda(), min(A.removal_bounds(n)[0], n), states)
    st_h = states.cpu().numpy()
    for j in range(12):
        g = I.philox(905, i, j)
        po, pl, removed = DO.destroy(inst, dec["ops"][j], dec["lens"][j], names[j], qs[j], g)
        nr = int(r["nremoved"][j])
        assert list(r["removed"][j, :nr].cpu().numpy()) == removed, (names[j], j)
        np.testing.assert_array_equal(r["lens"][j].cpu().numpy(), pl)
        np.testing.assert_array_equal(r["ops"][j].cpu().numpy(), po)
        assert np.array_equal(st_h[j], R.state_bytes(g)), (names[j], j)
