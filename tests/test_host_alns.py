"""Host-side ALNS pieces against the reference: the destroy oracle (the
checker of K6) against the reference's destroy goldens, the formulas, and the
construction helpers."""
import numpy as np
import pytest

import inputs as I
from conftest import config_instance
from paper_2602_23685_b200 import alns as A
from oracle import destroy_oracle as DO

CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


def test_oracle_destroy_matches_reference_goldens(golden, golden_meta):
    """oracle/destroy_oracle.py (the CPU restatement the K6 tests check
    against) reproduces the reference's destroy goldens for all six operators:
    removed set, partial solution and final generator state."""
    seen = set()
    for i, rec in enumerate(golden_meta["destroys"]):
        inst = config_instance(rec["key"])
        ops, lens = golden[f"{rec['key']}/dec_ops"][rec["case"]], golden[f"{rec['key']}/dec_lens"][rec["case"]]
        rng = I.philox(41, CID[rec["key"]], rec["case"])
        po, pl, removed = DO.destroy(inst, ops, lens, rec["operator"], rec["q"], rng)
        assert removed == list(golden[f"destroy/{i}/removed"]), rec
        np.testing.assert_array_equal(pl, golden[f"destroy/{i}/lens"])
        np.testing.assert_array_equal(po, golden[f"destroy/{i}/ops"][:2 * inst.n])
        st = rng.bit_generator.state
        assert [int(x) for x in st["state"]["counter"]] == rec["final_counter"]
        assert int(st["buffer_pos"]) == rec["final_buffer_pos"]
        assert int(st["has_uint32"]) == rec["final_has_uint32"]
        seen.add(rec["operator"])
    assert seen == set(A.DESTROY_OPERATORS)


def test_formulas():  # test_alns.py:18-45
    assert A.removal_bounds(80) == (4, 4)
    assert A.removal_bounds(202) == (5, 10)
    assert A.removal_bounds(431) == (10, 21)
    bank = A.OperatorBank.fresh()
    bank.weights["random"], bank.scores["random"], bank.attempts["random"] = 1.0, 33.0, 1
    bank.weights["worst"], bank.scores["worst"], bank.attempts["worst"] = 0.1, 0.0, 5
    bank.weights["shaw"], bank.attempts["shaw"] = 2.0, 0
    A.update_weights(bank, r=0.1)
    assert bank.weights["random"] == pytest.approx(4.2)
    assert bank.weights["worst"] == pytest.approx(0.1)
    assert bank.weights["shaw"] == pytest.approx(1.8)

    class Fixed:
        def __init__(self, v):
            self.v = v

        def random(self):
            return self.v
    import math
    assert A.sa_accept(90, 100, 10.0, Fixed(0.999))
    assert A.sa_accept(110, 100, 10.0, Fixed(math.exp(-1) - 1e-6))
    assert not A.sa_accept(110, 100, 10.0, Fixed(math.exp(-1) + 1e-6))
    with pytest.raises(ValueError):
        A.sa_accept(1, 2, 0.0, Fixed(0.5))


def test_sweep_order_is_permutation():
    inst = config_instance("eil51")
    order = A.sweep_order(inst)
    assert sorted(order) == list(inst.customers)


def test_sweep_and_balance_match_reference_rules():
    """sweep_order / _balance_sectors (numpy) against a direct statement of
    the reference's rules (alns.py:290-327) on every config instance."""
    from conftest import CONFIG_KEYS
    for key in CONFIG_KEYS:
        inst = config_instance(key)
        d, p = inst.arrays()
        cs = list(range(1, inst.n + 1))
        a = max(cs, key=lambda c: (d[0][c], -c))
        b = max(cs, key=lambda c: (d[a][c], -c))
        assert A.sweep_order(inst) == sorted(cs, key=lambda c: (d[a][c] - d[b][c], d[0][c], c))
        order = A.sweep_order(inst)
        sectors = [order[v::inst.m] if v % 2 else order[v * len(order) // inst.m:(v + 1) * len(order) // inst.m]
                   for v in range(inst.m)]
        w = {c: 2.0 * d[0][c] + p[c] for c in cs}
        secs = [list(x) for x in sectors]
        loads = [sum(w[c] for c in x) for x in secs]
        mean = sum(loads) / len(loads)
        for _ in range(2 * inst.n):
            if mean <= 0 or max(abs(x - mean) for x in loads) < 0.10 * mean:
                break
            hi = max(range(len(loads)), key=lambda i: loads[i])
            lo = min(range(len(loads)), key=lambda i: loads[i])
            if not secs[hi]:
                break
            bc, bp = None, max(loads)
            for c in secs[hi]:
                pk = max(loads[hi] - w[c], loads[lo] + w[c], *(loads[i] for i in range(len(loads)) if i not in (hi, lo)))
                if pk < bp:
                    bc, bp = c, pk
            if bc is None:
                break
            secs[hi].remove(bc)
            secs[lo].append(bc)
            loads[hi] -= w[bc]
            loads[lo] += w[bc]
        assert A._balance_sectors(inst, sectors) == secs, key
