"""Multi-rank ALNS pools (alns.run_pool_distributed): the
cross-rank global-share synchronisation on gloo, world size 2 (CPU), and a
whole sharded pool run (GPU, both ranks on cuda:0 over gloo: the ranks'
kernels never wait on one another)."""
import pytest

from test_islands_gloo import run_world


def _share_case(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from conftest import config_instance
    from paper_2602_23685_b200 import alns as A
    from paper_2602_23685_b200.schedule import Solution
    inst = config_instance("gr17")
    n = inst.n
    # rank r holds a distinct solution: customers split round-robin over vehicles
    tours = [[] for _ in range(inst.m)]
    for c in range(1, n + 1):
        v = (c + rank) % inst.m
        tours[v] += [(c, A._D), (c, A._P)]
    sol = Solution.from_lists(tours)
    out = {}
    s = A._PoolShare()
    A.sync_pool_share(inst, s, None)  # empty everywhere: untouched
    out["empty"] = (s.best_z, s.best_sol)
    s.offer(3, 100.0, sol)
    A.sync_pool_share(inst, s, None)  # tie: lowest rank wins
    out["tie"] = (s.best_z, s.src, s.best_sol.to_arrays(n)[0].tolist())
    s = A._PoolShare()
    s.offer(3, 90.0 if rank == 1 else 95.0, sol)
    A.sync_pool_share(inst, s, None)
    out["strict"] = (s.best_z, s.best_sol.to_arrays(n)[0].tolist())
    s = A._PoolShare()
    if rank == 1:
        s.offer(0, 50.0, sol)
    A.sync_pool_share(inst, s, None)  # only one rank has anything
    out["one"] = (s.best_z, s.best_sol.to_arrays(n)[0].tolist())
    own = sol.to_arrays(n)[0].tolist()
    return out, own


def test_sync_pool_share_world2():
    out = run_world(_share_case)
    (o0, own0), (o1, own1) = out[0], out[1]
    assert own0 != own1
    for o in (o0, o1):
        assert o["empty"] == (float("inf"), None)
        assert o["tie"] == (100.0, None, own0)
        assert o["strict"] == (90.0, own1)
        assert o["one"] == (50.0, own1)


def _pool_case(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch
    torch.cuda.set_device(0)
    from conftest import config_instance
    from paper_2602_23685_b200 import alns as A
    from paper_2602_23685_b200.schedule import evaluate
    inst = config_instance("eil51")
    params = A.AlnsParams(max_iter=40, workers_per_pool=3, pool_sync_interval=10, best_check_interval=10,
                          pickup_reposition_interval=20, cross_agent_interval=10**6)
    init = A.construct_initial(inst)
    best, info = A.run_pool_distributed(inst, params, pool_size=12, seed=5, initial=init)
    z = evaluate(inst, best).makespan
    local_best = min(st.best_trace[-1][1] for st in info["worker_stats"])
    return (z, info["best_makespan"], info["local_workers"], local_best, best.to_arrays(inst.n)[0].tolist())


@pytest.mark.gpu
def test_run_pool_distributed_world2_on_one_gpu():
    out = run_world(_pool_case)
    (z0, b0, n0, l0, s0), (z1, b1, n1, l1, s1) = out[0], out[1]
    assert n0 + n1 == 12 and n0 == 6
    assert z0 == z1 == b0 == b1 and s0 == s1  # every rank returns the global best
    assert z0 <= min(l0, l1)


def _pipeline_case(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch
    torch.cuda.set_device(0)
    from conftest import config_instance
    from paper_2602_23685_b200.pipeline import run_pipeline_budget_distributed
    from paper_2602_23685_b200.schedule import evaluate
    from paper_2602_23685_b200 import alns as A
    calls = []
    orig = A.sync_pool_share

    def counted(*a, **k):
        calls.append(1)
        return orig(*a, **k)
    A.sync_pool_share = counted
    inst = config_instance("gr17")
    sol, z, trace = run_pipeline_budget_distributed(inst, seconds=3.0, pool_size=8)
    return (z, evaluate(inst, sol).makespan, min(b for _, b in trace), sol.to_arrays(inst.n)[0].tolist(),
            len(calls))


@pytest.mark.gpu
def test_pipeline_budget_distributed_world2_on_one_gpu():
    out = run_world(_pipeline_case)
    (z0, e0, own0, s0, c0), (z1, e1, own1, s1, c1) = out[0], out[1]
    assert z0 == z1 == e0 == e1 and s0 == s1  # one global best everywhere
    assert z0 == min(own0, own1)
    # the ranks cooperate during the budget: the same number of incumbent
    # exchanges on both (stage boundaries + every kick round + the final one)
    assert c0 == c1 >= 4
