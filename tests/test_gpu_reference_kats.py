"""The reference's own known-answer tests, run through this package's public
API on the GPU (pkg/tests/test_schedule.py, test_brkga.py)."""
import numpy as np
import pytest

from paper_2602_23685_b200.instance import FleetConfig, Instance
from paper_2602_23685_b200.schedule import (CapacityViolation, Deadlock, MalformedSolution,
                                            ScheduleError, Solution, coordination_metrics,
                                            evaluate, exact_makespan, makespan,
                                            two_pass_estimate)

pytestmark = pytest.mark.gpu
D, P = "D", "P"


@pytest.fixture
def toy():
    return Instance(n=2, d=((0, 10, 12), (10, 0, 5), (12, 5, 0)), p=(0, 20, 20),
                    fleet=FleetConfig(1, 2), label="toy")


@pytest.fixture
def cross_toy():
    return Instance(n=1, d=((0, 10), (10, 0)), p=(0, 20), fleet=FleetConfig(2, 1), label="x")


@pytest.fixture
def single_toy():
    return Instance(n=1, d=((0, 10), (10, 0)), p=(0, 20), fleet=FleetConfig(1, 1), label="s")


def test_single_vehicle_drop_wait_pick(single_toy):  # test_schedule.py:16-20
    sched = evaluate(single_toy, Solution.from_lists([[(1, D), (1, P)]]))
    assert sched.t_drop[1] == 10 and sched.t_pickup[1] == 30 and sched.makespan == 40


def test_interleaved_single_route(toy):  # test_schedule.py:23-27
    sched = evaluate(toy, Solution.from_lists([[(1, D), (2, D), (1, P), (2, P)]]))
    assert sched.t_drop == {1: 10, 2: 15}
    assert sched.t_pickup == {1: 30, 2: 35}
    assert sched.makespan == 47
    assert makespan(sched) == 47
    assert exact_makespan(toy, Solution.from_lists([[(1, D), (2, D), (1, P), (2, P)]])) == 47


def test_cross_vehicle_precedence(cross_toy):  # test_schedule.py:30-35
    sched = evaluate(cross_toy, Solution.from_lists([[(1, D)], [(1, P)]]))
    assert sched.returns == [20, 40] and sched.makespan == 40 and sched.t_pickup[1] == 30
    assert sched.bottleneck() == 1


def test_empty_route_returns_zero():  # test_schedule.py:38-46
    inst = Instance(n=1, d=((0, 1), (1, 0)), p=(0, 0), fleet=FleetConfig(2, 1), label="e")
    sched = evaluate(inst, Solution.from_lists([[(1, D), (1, P)], []]))
    assert sched.returns[1] == 0.0


def test_estimates(toy, cross_toy):  # test_schedule.py:86-101
    assert two_pass_estimate(toy, Solution.from_lists([[(1, D), (2, D), (1, P), (2, P)]])) == 47
    assert two_pass_estimate(cross_toy, Solution.from_lists([[(1, D)], [(1, P)]])) == 40
    sol = Solution.from_lists([[(2, D), (2, P), (1, D), (1, P)]])
    assert two_pass_estimate(toy, sol) == 47
    assert evaluate(toy, sol).makespan == 67
    assert exact_makespan(toy, sol) == 67


def test_error_classes(single_toy):  # test_schedule.py:106-146
    k1 = Instance(n=2, d=((0, 10, 12), (10, 0, 5), (12, 5, 0)), p=(0, 20, 20),
                  fleet=FleetConfig(1, 1), label="k1")
    sol = Solution.from_lists([[(1, D), (2, D), (1, P), (2, P)]])
    for fn in (evaluate, exact_makespan, two_pass_estimate):
        with pytest.raises(CapacityViolation):
            fn(k1, sol)
    k1b = Instance(n=2, d=k1.d, p=k1.p, fleet=FleetConfig(2, 1), label="k1b")
    with pytest.raises(CapacityViolation):
        evaluate(k1b, Solution.from_lists([[(1, D), (2, D)], [(1, P), (2, P)]]))
    for fn in (evaluate, exact_makespan, two_pass_estimate):
        with pytest.raises(Deadlock):
            fn(single_toy, Solution.from_lists([[(1, P), (1, D)]]))
    cyc = Instance(n=2, d=((0, 5, 5), (5, 0, 5), (5, 5, 0)), p=(0, 10, 10),
                   fleet=FleetConfig(2, 5), label="cyc")
    with pytest.raises(Deadlock):
        evaluate(cyc, Solution.from_lists([[(1, P), (2, D)], [(2, P), (1, D)]]))
    with pytest.raises(Deadlock):
        exact_makespan(cyc, Solution.from_lists([[(1, P), (2, D)], [(2, P), (1, D)]]))
    with pytest.raises(MalformedSolution):
        evaluate(single_toy, Solution.from_lists([[(1, D)]]))
    with pytest.raises(MalformedSolution):
        evaluate(single_toy, Solution.from_lists([[(1, D), (1, D), (1, P)]]))
    with pytest.raises(MalformedSolution):
        evaluate(single_toy, Solution.from_lists([[(1, D), (1, P)], []]))


def test_coordination_metrics(toy, cross_toy):  # test_schedule.py:51-81
    sol = Solution.from_lists([[(1, D)], [(1, P)]])
    assert coordination_metrics(cross_toy, sol, evaluate(cross_toy, sol)).cross_agent_pct == 100.0
    sol = Solution.from_lists([[(1, D), (2, D), (1, P), (2, P)]])
    m = coordination_metrics(toy, sol, evaluate(toy, sol))
    assert m.interleaved_pct == 100.0 and m.cross_agent_pct == 0.0


def test_schedule_rows_export(toy):  # test_schedule.py:157-163
    rows = evaluate(toy, Solution.from_lists([[(1, D), (2, D), (1, P), (2, P)]])).to_rows()
    assert len(rows) == 4
    assert rows[0] == {"vehicle": 0, "seq": 0, "customer": 1, "op": "D", "arrival": 10,
                       "time": 10, "q_after": 1}


def test_exact_equals_evaluate_on_random_solutions():  # test_schedule.py:194-204 property
    import inputs as I
    rng = np.random.default_rng(0)
    for trial in range(60):
        n = int(rng.integers(1, 7))
        m, k = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        pts = rng.integers(0, 80, size=(n + 1, 2))
        d = [[float(round(np.hypot(*(pts[i] - pts[j])))) for j in range(n + 1)] for i in range(n + 1)]
        p = [0.0] + [float(x) for x in rng.integers(20, 120, n)]
        inst = Instance.from_arrays(np.array(d), np.array(p), m, k, label="h")
        ops, lens = I.random_candidates(n, m, 1, (trial, 77))
        sol = Solution.from_arrays(ops[0], lens[0])
        try:
            z = evaluate(inst, sol).makespan
        except ScheduleError:
            with pytest.raises(ScheduleError):
                exact_makespan(inst, sol)
            continue
        assert exact_makespan(inst, sol) == z
