"""two_opt_improve on the device (baselines.py, vrp_ls_build kinds 2/0/3 +
K1 evaluate) against the reference's own results -- identical for any chunk
size, since only the first improving candidate of a scan is ever taken."""
import numpy as np
import pytest

from conftest import config_instance
from paper_2602_23685_b200 import baselines as BL
from paper_2602_23685_b200.schedule import Solution, evaluate

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunk", [BL.CHUNK, 13, 1])
def test_two_opt_improve_matches_reference(chunk, golden, golden_meta):
    for i, rec in enumerate(golden_meta["polish"]):
        if chunk == 1 and rec["key"] != "gr17":
            continue  # one candidate per launch: the sequential reference loop, kept small
        inst = config_instance(rec["key"])
        sol = Solution.from_arrays(golden[f"{rec['key']}/dec_ops"][rec["case"]],
                                   golden[f"{rec['key']}/dec_lens"][rec["case"]])
        out = BL.two_opt_improve(inst, sol, move_budget=rec["budget"], chunk=chunk)
        ops, lens = out.to_arrays(inst.n)
        np.testing.assert_array_equal(lens, golden[f"polish/{i}/lens"], err_msg=f"{i} chunk={chunk}")
        np.testing.assert_array_equal(ops, golden[f"polish/{i}/ops"], err_msg=f"{i} chunk={chunk}")
        assert evaluate(inst, out).makespan <= evaluate(inst, sol).makespan
