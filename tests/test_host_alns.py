"""Host-side ALNS pieces against the reference: removal cascade, destroy
operators that need no schedule (random / worst / cluster / route), formulas."""
import numpy as np
import pytest

import inputs as I
from conftest import config_instance
from paper_2602_23685_b200 import alns as A
from paper_2602_23685_b200 import insertion as INS
from paper_2602_23685_b200.schedule import Solution

CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


def test_remove_customers_matches_reference(golden, golden_meta):
    for i, rec in enumerate(golden_meta["repairs"]):
        inst = config_instance(rec["key"])
        sol = Solution.from_arrays(golden[f"{rec['key']}/dec_ops"][rec["case"]],
                                   golden[f"{rec['key']}/dec_lens"][rec["case"]])
        tours, removed = INS.remove_customers(inst, sol, [int(x) for x in golden[f"repair/{i}/pick"]])
        assert removed == list(golden[f"repair/{i}/removed"])
        ops, lens = Solution.from_lists(tours).to_arrays(inst.n)
        np.testing.assert_array_equal(lens, golden[f"repair/{i}/partial_lens"])
        np.testing.assert_array_equal(ops, golden[f"repair/{i}/partial_ops"])


def check_destroy(golden, golden_meta, operators):
    seen = 0
    for i, rec in enumerate(golden_meta["destroys"]):
        if rec["operator"] not in operators:
            continue
        inst = config_instance(rec["key"])
        sol = Solution.from_arrays(golden[f"{rec['key']}/dec_ops"][rec["case"]],
                                   golden[f"{rec['key']}/dec_lens"][rec["case"]])
        rng = I.philox(41, CID[rec["key"]], rec["case"])
        partial, removed = A.destroy(inst, sol, rec["operator"], rec["q"], rng)
        assert removed == list(golden[f"destroy/{i}/removed"]), rec
        ops, lens = partial.to_arrays(inst.n)
        np.testing.assert_array_equal(lens, golden[f"destroy/{i}/lens"])
        np.testing.assert_array_equal(ops, golden[f"destroy/{i}/ops"])
        st = rng.bit_generator.state
        assert [int(x) for x in st["state"]["counter"]] == rec["final_counter"]
        assert int(st["buffer_pos"]) == rec["final_buffer_pos"]
        assert int(st["has_uint32"]) == rec["final_has_uint32"]
        seen += 1
    assert seen


def test_destroy_without_schedule_matches_reference(golden, golden_meta):
    check_destroy(golden, golden_meta, ("random", "worst", "cluster", "route"))


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
