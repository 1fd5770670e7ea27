"""Device-resident ALNS (csrc/alns_step.cu): K6 destroy against the
reference's destroy goldens and the host destroy at scale, and whole
vrp_alns_iterate trajectories against the reference's run_alns goldens and
the host engine (pools included)."""
import numpy as np
import pytest
import torch

import inputs as I
from conftest import config_instance
from oracle import destroy_oracle as DO
from oracle import oracle as O
from paper_2602_23685_b200 import alns as A
from paper_2602_23685_b200 import device as DV
from paper_2602_23685_b200 import rng as R
from paper_2602_23685_b200.schedule import Solution

pytestmark = pytest.mark.gpu
CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


def _destroy_dev(inst, sols, ops_names, qs, gens):
    n = inst.n
    arrs = [s.to_arrays(n) for s in sols]
    ops = np.stack([o[:2 * n] for o, _ in arrs])
    lens = np.stack([l for _, l in arrs])
    states = torch.from_numpy(np.stack([R.state_bytes(g) for g in gens])).cuda()
    codes = np.array([DV.DESTROY_CODES[o] for o in ops_names], np.int32)
    r = DV.destroy_batch(inst, torch.from_numpy(ops).cuda(), torch.from_numpy(lens).cuda(),
                         torch.from_numpy(codes).cuda(), torch.from_numpy(np.asarray(qs, np.int32)).cuda(),
                         min(A.removal_bounds(n)[0], n), states)
    st = states.cpu().numpy()
    for g, raw in zip(gens, st):
        R.set_state_bytes(g, raw)
    nr = r["nremoved"].cpu().numpy()
    rem = r["removed"].cpu().numpy()
    return r["ops"].cpu().numpy(), r["lens"].cpu().numpy(), [list(rem[i, :nr[i]]) for i in range(len(sols))]


def test_destroy_kernel_matches_reference_goldens(golden, golden_meta):
    by_key = {}
    for i, rec in enumerate(golden_meta["destroys"]):
        by_key.setdefault(rec["key"], []).append(i)
    for key, idx in by_key.items():
        inst = config_instance(key)
        recs = [golden_meta["destroys"][i] for i in idx]
        sols = [Solution.from_arrays(golden[f"{key}/dec_ops"][r["case"]], golden[f"{key}/dec_lens"][r["case"]])
                for r in recs]
        gens = [I.philox(41, CID[key], r["case"]) for r in recs]
        o, l, rem = _destroy_dev(inst, sols, [r["operator"] for r in recs], [r["q"] for r in recs], gens)
        for j, (i, r) in enumerate(zip(idx, recs)):
            msg = f"{key} {r['operator']} case {r['case']}"
            assert rem[j] == list(golden[f"destroy/{i}/removed"]), msg
            np.testing.assert_array_equal(l[j], golden[f"destroy/{i}/lens"], err_msg=msg)
            np.testing.assert_array_equal(o[j], golden[f"destroy/{i}/ops"], err_msg=msg)
            st = gens[j].bit_generator.state
            assert [int(x) for x in st["state"]["counter"]] == r["final_counter"], msg
            assert int(st["buffer_pos"]) == r["final_buffer_pos"], msg
            assert int(st["has_uint32"]) == r["final_has_uint32"], msg


@pytest.mark.parametrize("key,count", [("gr17", 48), ("eil51", 48), ("kroA100", 36), ("a280", 18),
                                       ("dsj1000", 6)])
def test_destroy_kernel_vs_host_at_scale(key, count, golden):
    """K6 against the destroy oracle: fresh seeds; every operator; q across [q_min, q_max]."""
    inst = config_instance(key)
    n = inst.n
    base = golden[f"{key}/dec_ops"], golden[f"{key}/dec_lens"]
    qmin, qmax = A.removal_bounds(n)
    sols, names, qs = [], [], []
    for i in range(count):
        j = i % base[0].shape[0]
        sols.append(Solution.from_arrays(base[0][j], base[1][j]))
        names.append(A.DESTROY_OPERATORS[i % 6])
        qs.append(min(n, qmin + (i * 7) % (qmax - qmin + 1) + (i % 5 == 4) * 3))
    g_dev = [I.philox(71, CID[key], i) for i in range(count)]
    o, l, rem = _destroy_dev(inst, sols, names, qs, g_dev)
    for i in range(count):
        g = I.philox(71, CID[key], i)
        po, pl, removed = DO.destroy(inst, base[0][i % base[0].shape[0]], base[1][i % base[0].shape[0]],
                                     names[i], qs[i], g)
        assert rem[i] == removed, (names[i], i)
        np.testing.assert_array_equal(l[i], pl, err_msg=f"{names[i]} {i}")
        np.testing.assert_array_equal(o[i], po, err_msg=f"{names[i]} {i}")
        assert np.array_equal(R.state_bytes(g), R.state_bytes(g_dev[i])), (names[i], i)


def test_device_run_alns_matches_reference(golden, golden_meta):
    for j, run in enumerate(golden_meta["alns_runs"]):
        inst = config_instance(run["key"])
        params = A.AlnsParams(max_iter=run["iters"], **run["extra"])
        initial = None
        if run["init"]:
            initial = Solution.from_arrays(golden[f"{run['key']}/dec_ops"][0],
                                           golden[f"{run['key']}/dec_lens"][0])
        best, st = A.run_alns(inst, params, seed=run["seed"], initial=initial, engine="device")
        ops, lens = best.to_arrays(inst.n)
        np.testing.assert_array_equal(ops, golden[f"alns/{j}/ops"], err_msg=str(j))
        np.testing.assert_array_equal(lens, golden[f"alns/{j}/lens"])
        assert [list(x) for x in st.best_trace] == [list(x) for x in run["best_trace"]], j
        assert st.accepted == run["accepted"] and st.rejected_candidates == run["rejected"], j
        assert st.reheats == run["reheats"]
        assert st.final_temperature == run["final_temperature"]
        assert st.attempts == run["attempts"]
        assert st.weight_rows == run["weight_rows"], j


def _same_stats(a, b):
    assert a.best_trace == b.best_trace
    assert a.accepted == b.accepted and a.rejected_candidates == b.rejected_candidates
    assert a.reheats == b.reheats and a.final_temperature == b.final_temperature
    assert a.attempts == b.attempts and a.weight_rows == b.weight_rows


@pytest.mark.parametrize("key,iters,seed", [("eil51", 450, 3), ("kroA100", 120, 4), ("a280", 25, 5),
                                            ("dsj1000", 4, 6)])
def test_device_engine_equals_host_engine(key, iters, seed):
    """Longer single trajectories (local search at 200/400 included)."""
    inst = config_instance(key)
    params = A.AlnsParams(max_iter=iters, weight_interval=40, stagnation_threshold=30, t0=0.05)
    initial = A.construct_initial(inst)
    b1, s1 = A.run_alns(inst, params, seed=seed, initial=initial, engine="device")
    b2, s2 = A.run_alns(inst, params, seed=seed, initial=initial, engine="host")
    assert b1 == b2
    _same_stats(s1, s2)


def test_device_pool_equals_host_pool():
    """Pools with share polling / merging at stretch boundaries."""
    inst = config_instance("eil51")
    params = A.AlnsParams(max_iter=60, best_check_interval=7, pool_sync_interval=5, workers_per_pool=3,
                          pickup_reposition_interval=20, cross_agent_interval=50)
    initial = A.construct_initial(inst)
    b1, i1 = A.run_pool(inst, params, pool_size=8, seed=21, initial=initial, engine="device")
    b2, i2 = A.run_pool(inst, params, pool_size=8, seed=21, initial=initial, engine="host")
    assert b1 == b2 and i1["best_makespan"] == i2["best_makespan"]
    for a, b in zip(i1["worker_stats"], i2["worker_stats"]):
        _same_stats(a, b)


def test_device_engine_equals_host_engine_fractional_instance():
    """alns_kernel<false,false> (fp64 distances, one-lane passes): the device
    engine equals the host engine on a non-integral instance."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("eil51")
    d, p = base.arrays()
    g = np.random.default_rng(21)
    d2 = d + g.random(d.shape) * 0.7
    d2 = (d2 + d2.T) / 2
    np.fill_diagonal(d2, 0.0)
    p2 = p + g.random(p.shape) / 3
    p2[0] = 0.0
    inst = Instance.from_arrays(d2, p2, base.m, base.k, label="eil51-frac")
    params = A.AlnsParams(max_iter=60, weight_interval=20, stagnation_threshold=15, t0=0.05)
    initial = A.construct_initial(inst)
    b1, s1 = A.run_alns(inst, params, seed=8, initial=initial, engine="device")
    b2, s2 = A.run_alns(inst, params, seed=8, initial=initial, engine="host")
    assert b1 == b2
    _same_stats(s1, s2)


def test_sa_exp_correctly_rounded():
    """The SA threshold exp (alns.py:588) that vrp_alns_iterate uses is the
    correctly rounded fp64 exp: checked against 50-digit decimal exp."""
    import decimal
    from paper_2602_23685_b200 import _native as N
    decimal.getcontext().prec = 50
    g = np.random.default_rng(9)
    x = np.concatenate([-g.random(40000) * 40, g.uniform(-700, 700, 4000), -g.random(2000) * 1e-6,
                        [0.0, -0.5, -1.0, -707.9, 708.9]])
    want = np.array([float(decimal.Decimal(float(v)).exp()) for v in x])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    N.check(N.lib().vrp_sa_exp(N.ptr(xd), N.ptr(yd), x.size, N.stream_handle()), "vrp_sa_exp")
    np.testing.assert_array_equal(yd.cpu().numpy(), want)


def test_reference_signature_destroy_and_removal_api(golden, golden_meta):
    """The drop-in signatures run K6 on the device: alns.destroy (batch of
    one, the caller's Philox generator round-tripped) equals the reference's
    destroy goldens; insertion.remove_customers equals the repair goldens'
    partials; insertion.removal_gains equals the oracle's."""
    from paper_2602_23685_b200 import insertion as INS
    for i, rec in enumerate(golden_meta["destroys"]):
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
    for i, rec in enumerate(golden_meta["repairs"]):
        inst = config_instance(rec["key"])
        sol = Solution.from_arrays(golden[f"{rec['key']}/dec_ops"][rec["case"]],
                                   golden[f"{rec['key']}/dec_lens"][rec["case"]])
        tours, removed = INS.remove_customers(inst, sol, [int(x) for x in golden[f"repair/{i}/pick"]])
        assert removed == list(golden[f"repair/{i}/removed"])
        ops, lens = Solution.from_lists(tours).to_arrays(inst.n)
        np.testing.assert_array_equal(lens, golden[f"repair/{i}/partial_lens"])
        np.testing.assert_array_equal(ops, golden[f"repair/{i}/partial_ops"])
    for key in ("gr17", "eil51", "kroA100", "a280", "dsj1000"):
        inst = config_instance(key)
        for j in range(2):
            o, l = golden[f"{key}/dec_ops"][j], golden[f"{key}/dec_lens"][j]
            gains = INS.removal_gains(inst, Solution.from_arrays(o, l))
            want = DO.removal_gains(inst, o, l)
            assert [gains[c] for c in inst.customers] == list(want[1:]), key


def test_removal_api_on_partial_solutions(golden):
    """insertion.removal_gains / remove_customers (K6 device code) on partial
    solutions -- customers absent from every route -- against the oracle."""
    from paper_2602_23685_b200 import insertion as INS
    for key in ("eil51", "a280", "dsj1000"):
        inst = config_instance(key)
        o, l = golden[f"{key}/dec_ops"][1], golden[f"{key}/dec_lens"][1]
        pick = I.philox(91, CID[key]).choice(np.arange(1, inst.n + 1), size=5, replace=False)
        po, pl, rem = O.remove_customers(inst, o, l, pick)
        part = Solution.from_arrays(po, pl)
        gains = INS.removal_gains(inst, part)
        want = DO.removal_gains(inst, po, pl)
        assert [gains[c] for c in inst.customers] == list(want[1:]), key
        more = I.philox(92, CID[key]).choice(np.setdiff1d(np.arange(1, inst.n + 1), rem), size=3, replace=False)
        tours, removed = INS.remove_customers(inst, part, [int(c) for c in more])
        wo, wl, wr = O.remove_customers(inst, po, pl, more)
        assert removed == [int(c) for c in wr], key
        to, tl = Solution.from_lists(tours).to_arrays(inst.n)
        np.testing.assert_array_equal(tl, wl)
        np.testing.assert_array_equal(to[:int(tl.sum())], wo[:int(wl.sum())])


@pytest.mark.parametrize("m,k,n_nodes", [(2, 6, 90), (12, 3, 160)])
def test_team_alns_engine_other_fleet_shapes(m, k, n_nodes):
    """vrp_alns_iterate's CTA-per-worker path on fleets other than m = 6:
    the device engine equals the host engine (K6 + batched K5 + K1 + host
    acceptance)."""
    from paper_2602_23685_b200.instance import Instance
    g = np.random.default_rng(m * 100 + k)
    pts = g.integers(0, 500, size=(n_nodes, 2))
    d = np.ceil(np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)))
    p = np.concatenate([[0.0], g.integers(5, 400, size=n_nodes - 1).astype(float)])
    inst = Instance.from_arrays(d, p, m, k, label=f"team-alns-m{m}")
    params = A.AlnsParams(max_iter=12, weight_interval=5, stagnation_threshold=4, t0=0.05,
                          pickup_reposition_interval=10**6, cross_agent_interval=10**6)
    initial = A.construct_initial(inst)
    b1, s1 = A.run_alns(inst, params, seed=9, initial=initial, engine="device")
    b2, s2 = A.run_alns(inst, params, seed=9, initial=initial, engine="host")
    assert b1 == b2
    _same_stats(s1, s2)
