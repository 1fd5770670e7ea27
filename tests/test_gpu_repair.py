"""GPU parity of K5 (ALNS repair, insertion.reinsert_all) against the
reference's goldens and, at scale, against the oracle -- repaired tours,
RepairFailed status and the final generator state must all match."""
import numpy as np
import pytest

import inputs as I
from conftest import config_instance
from oracle import oracle as O
from paper_2602_23685_b200 import insertion as INS

pytestmark = pytest.mark.gpu
CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


def same_state(a, b):
    sa, sb = a.bit_generator.state, b.bit_generator.state
    return (np.array_equal(sa["state"]["counter"], sb["state"]["counter"])
            and np.array_equal(sa["buffer"], sb["buffer"]) and sa["buffer_pos"] == sb["buffer_pos"]
            and sa["has_uint32"] == sb["has_uint32"] and sa["uinteger"] == sb["uinteger"])


def test_repair_matches_reference_goldens(golden, golden_meta):
    recs = golden_meta["repairs"]
    by_key = {}
    for i, rec in enumerate(recs):
        by_key.setdefault(rec["key"], []).append(i)
    for key, idx in by_key.items():
        inst = config_instance(key)
        ops = np.stack([golden[f"repair/{i}/partial_ops"] for i in idx])
        lens = np.stack([golden[f"repair/{i}/partial_lens"] for i in idx])
        removed = [golden[f"repair/{i}/removed"] for i in idx]
        rks = [recs[i]["regret_k"] for i in idx]
        with_rng = [i for i in idx if recs[i]["rng"]]
        without = [i for i in idx if not recs[i]["rng"]]
        for group, use in ((with_rng, True), (without, False)):
            if not group:
                continue
            sel = [idx.index(i) for i in group]
            gens = [I.philox(37, CID[key], recs[i]["case"]) for i in group] if use else None
            o, l, st = INS.reinsert_batch(inst, ops[sel], lens[sel], [removed[j] for j in sel],
                                          [rks[j] for j in sel], gens)
            for j, i in enumerate(group):
                assert st[j] == recs[i]["status"], (key, i)
                np.testing.assert_array_equal(l[j], golden[f"repair/{i}/lens"], err_msg=f"{key} {i}")
                np.testing.assert_array_equal(o[j], golden[f"repair/{i}/ops"], err_msg=f"{key} {i}")
                if use:
                    s = gens[j].bit_generator.state
                    assert [int(x) for x in s["state"]["counter"]] == recs[i]["final_counter"]
                    assert int(s["buffer_pos"]) == recs[i]["final_buffer_pos"]
                    assert int(s["has_uint32"]) == recs[i]["final_has_uint32"]


@pytest.mark.parametrize("key,count,q", [("gr17", 64, 6), ("eil51", 64, 8), ("kroA100", 32, 10),
                                         ("a280", 8, 14)])
def test_repair_batch_vs_oracle(key, count, q, golden):
    inst = config_instance(key)
    genes = I.chromosomes(inst.n, count, (61, CID[key]))
    dec = O.decode_batch(inst, genes)
    parts, plens, removed, rks = [], [], [], []
    for i in range(count):
        pick = I.philox(62, CID[key], i).choice(np.arange(1, inst.n + 1), size=q, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * inst.n])
        plens.append(l)
        removed.append(r)
        rks.append((0, 2, 3, inst.m)[i % 4])
    parts, plens = np.stack(parts), np.stack(plens)
    dev_gens = [I.philox(63, CID[key], i) for i in range(count)]
    o, l, st = INS.reinsert_batch(inst, parts, plens, removed, rks, dev_gens)
    for i in range(count):
        g = I.philox(63, CID[key], i)
        rst, ro, rl = O.reinsert_all(inst, parts[i], plens[i], removed[i], rks[i], g)
        assert st[i] == rst, i
        if rst == 0:
            np.testing.assert_array_equal(l[i], rl)
            np.testing.assert_array_equal(o[i], ro)
        assert same_state(dev_gens[i], g), i


def test_reinsert_all_api_toy():  # test_alns.py:107-116: the toy rebuilds to 47
    from paper_2602_23685_b200.instance import FleetConfig, Instance
    from paper_2602_23685_b200.schedule import evaluate
    toy = Instance(n=2, d=((0, 10, 12), (10, 0, 5), (12, 5, 0)), p=(0, 20, 20),
                   fleet=FleetConfig(1, 2), label="toy")
    ctx = INS.InsertionContext(toy, [[]])
    INS.reinsert_all(ctx, [1, 2], 0, np.random.Generator(np.random.Philox(key=(1, 1))))
    assert evaluate(toy, ctx.solution()).makespan == 47


def test_repair_non_integral_instance_vs_oracle():
    """fp64 instance (no exact-integer sums): K5 keeps the reference's
    left-to-right passes; integral instances take the warp-scan passes."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("kroA100")
    d, p = base.arrays()
    rng = np.random.default_rng(11)
    d2 = d + rng.random(d.shape) * 0.61
    d2 = (d2 + d2.T) / 2
    np.fill_diagonal(d2, 0.0)
    p2 = p * 1.0003 + rng.random(p.shape) / 7
    p2[0] = 0.0
    inst = Instance.from_arrays(d2, p2, base.m, base.k, label="kro-frac")
    count = 24
    dec = O.decode_batch(inst, I.chromosomes(inst.n, count, (64, 3)))
    parts, plens, removed, rks = [], [], [], []
    for i in range(count):
        pick = I.philox(65, 3, i).choice(np.arange(1, inst.n + 1), size=9, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * inst.n]); plens.append(l); removed.append(r)
        rks.append((0, 2, 3, inst.m)[i % 4])
    parts, plens = np.stack(parts), np.stack(plens)
    dev_gens = [I.philox(66, 3, i) for i in range(count)]
    o, l, st = INS.reinsert_batch(inst, parts, plens, removed, rks, dev_gens)
    for i in range(count):
        g = I.philox(66, 3, i)
        rst, ro, rl = O.reinsert_all(inst, parts[i], plens[i], removed[i], rks[i], g)
        assert st[i] == rst, i
        if rst == 0:
            np.testing.assert_array_equal(l[i], rl)
            np.testing.assert_array_equal(o[i], ro)
        assert same_state(dev_gens[i], g), i


def _dsj_cases():
    """16 repairs at the dsj1000 size (n = 999): block-structured solutions
    (route-local customers, so the removed set is exactly the q picked) with
    q in {2, 24, 49}, plus decoded solutions whose capacity cascade grows
    q = 2 to ~50 removed customers (insertion.py:379-397)."""
    inst = config_instance("dsj1000")
    n = inst.n
    blk_ops, blk_lens = I.block_candidates(n, inst.m, inst.k, 12, (71, 5, 0))
    dec = O.decode_batch(inst, I.chromosomes(n, 4, (71, 5)))
    srcs = [(blk_ops[i], blk_lens[i], (2, 24, 49)[i % 3]) for i in range(12)]
    srcs += [(dec["ops"][i], dec["lens"][i], 2) for i in range(4)]
    parts, plens, removed, rks = [], [], [], []
    for i, (ops, lens, q) in enumerate(srcs):
        pick = I.philox(72, 5, i).choice(np.arange(1, n + 1), size=q, replace=False)
        o, l, r = O.remove_customers(inst, ops, lens, pick)
        parts.append(o[:2 * n]); plens.append(l); removed.append(r)
        rks.append((0, 2, 3, inst.m)[i % 4])
    return inst, np.stack(parts), np.stack(plens), removed, rks


def test_repair_batch_vs_oracle_dsj1000():
    """K5 at n = 999 (the size the product runs it at, pipeline.py) against
    the oracle's reinsert_all: tours, RepairFailed and generator state;
    12 cases with a Generator(Philox) and 4 deterministic (rng=None)."""
    inst, parts, plens, removed, rks = _dsj_cases()
    assert sorted({len(r) for r in removed[:12]}) == [2, 24, 49]
    assert min(len(r) for r in removed[12:]) > 2  # the cascade fired
    with_rng = list(range(12))
    without = list(range(12, 16))
    for group, use in ((with_rng, True), (without, False)):
        gens = [I.philox(73, 5, i) for i in group] if use else None
        o, l, st = INS.reinsert_batch(inst, parts[group], plens[group], [removed[i] for i in group],
                                      [rks[i] for i in group], gens)
        for j, i in enumerate(group):
            g = I.philox(73, 5, i) if use else None
            rst, ro, rl = O.reinsert_all(inst, parts[i], plens[i], removed[i], rks[i], g)
            assert st[j] == rst, i
            if rst == 0:
                np.testing.assert_array_equal(l[j], rl, err_msg=str(i))
                np.testing.assert_array_equal(o[j], ro, err_msg=str(i))
            if use:
                assert same_state(gens[j], g), i


@pytest.mark.parametrize("m,k,n_nodes", [(1, 40, 80), (2, 6, 90), (12, 3, 160)])
def test_team_repair_other_fleet_shapes_vs_oracle(m, k, n_nodes):
    """The CTA-per-repair path (integral instances with 2n >= 24 m) on fleets
    other than the benchmark's m = 6: one vehicle, two, and twelve (more
    routes than a 8-lane segment), against the oracle's reinsert_all."""
    from paper_2602_23685_b200.instance import Instance
    g = np.random.default_rng(m * 100 + k)
    pts = g.integers(0, 500, size=(n_nodes, 2))
    d = np.ceil(np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)))
    p = np.concatenate([[0.0], g.integers(5, 400, size=n_nodes - 1).astype(float)])
    inst = Instance.from_arrays(d, p, m, k, label=f"team-m{m}")
    n = inst.n
    assert 2 * n >= 24 * m  # the team path
    count = 12
    dec = O.decode_batch(inst, I.chromosomes(n, count, (95, m)))
    parts, plens, removed, rks = [], [], [], []
    for i in range(count):
        pick = I.philox(96, m, i).choice(np.arange(1, n + 1), size=6, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * n]); plens.append(l); removed.append(r)
        rks.append((0, 2, 3, m)[i % 4] if m > 1 else 0)
    parts, plens = np.stack(parts), np.stack(plens)
    gens = [I.philox(97, m, i) for i in range(count)]
    o, l, st = INS.reinsert_batch(inst, parts, plens, removed, rks, gens)
    for i in range(count):
        gi = I.philox(97, m, i)
        rst, ro, rl = O.reinsert_all(inst, parts[i], plens[i], removed[i], rks[i], gi)
        assert st[i] == rst, i
        if rst == 0:
            np.testing.assert_array_equal(l[i], rl, err_msg=str(i))
            np.testing.assert_array_equal(o[i], ro, err_msg=str(i))
        assert same_state(gens[i], gi), i
