"""Pin the oracle's restatement of insertion.py (removal cascade, customer
options, greedy / regret reinsertion with the windowed RNG picks) to the
reference's own outputs (tests/golden, Generator(Philox) injected)."""
import numpy as np
import pytest

import inputs as I
from conftest import config_instance
from oracle import oracle as O

CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


def test_py_sum_matches_cpython():
    rng = np.random.default_rng(0)
    for _ in range(200):
        x = (rng.random(rng.integers(1, 9)) - 0.3) * 10.0 ** rng.integers(-3, 9)
        assert O.py_sum(x) == sum(x.tolist())
    assert O.py_sum([0.1] * 10) == 1.0


def test_remove_customers_matches_reference(golden, golden_meta):
    for i, rec in enumerate(golden_meta["repairs"]):
        inst = config_instance(rec["key"])
        tag = f"repair/{i}"
        base_ops = golden[f"{rec['key']}/dec_ops"][rec["case"]]
        base_lens = golden[f"{rec['key']}/dec_lens"][rec["case"]]
        ops, lens, removed = O.remove_customers(inst, base_ops, base_lens, golden[tag + "/pick"])
        np.testing.assert_array_equal(removed, golden[tag + "/removed"])
        np.testing.assert_array_equal(lens, golden[tag + "/partial_lens"])
        L = int(lens.sum())
        np.testing.assert_array_equal(ops[:L], golden[tag + "/partial_ops"][:L])


def test_reinsert_all_matches_reference(golden, golden_meta):
    for i, rec in enumerate(golden_meta["repairs"]):
        inst = config_instance(rec["key"])
        tag = f"repair/{i}"
        gen = I.philox(37, CID[rec["key"]], rec["case"]) if rec["rng"] else None
        st, ops, lens = O.reinsert_all(inst, golden[tag + "/partial_ops"], golden[tag + "/partial_lens"],
                                       golden[tag + "/removed"], rec["regret_k"], gen)
        assert st == rec["status"], i
        if st == 0:
            np.testing.assert_array_equal(lens, golden[tag + "/lens"], err_msg=str(rec))
            np.testing.assert_array_equal(ops, golden[tag + "/ops"], err_msg=str(rec))
        if gen is not None:
            s = gen.bit_generator.state
            assert [int(x) for x in s["state"]["counter"]] == rec["final_counter"], i
            assert int(s["buffer_pos"]) == rec["final_buffer_pos"]
            assert int(s["has_uint32"]) == rec["final_has_uint32"]
            assert int(s["uinteger"]) == rec["final_uinteger"]
