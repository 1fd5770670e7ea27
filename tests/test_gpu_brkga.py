"""GPU parity of the BRKGA generation step (K4) and the device-resident
run_brkga loop against the reference (goldens) and the oracle."""
import numpy as np
import pytest
import torch

import inputs as I
from conftest import config_instance
from oracle import oracle as O
from paper_2602_23685_b200 import brkga as B

pytestmark = pytest.mark.gpu


def same_state(a, b):
    sa, sb = a.bit_generator.state, b.bit_generator.state
    return (np.array_equal(sa["state"]["counter"], sb["state"]["counter"])
            and np.array_equal(sa["state"]["key"], sb["state"]["key"])
            and np.array_equal(sa["buffer"], sb["buffer"])
            and sa["buffer_pos"] == sb["buffer_pos"] and sa["has_uint32"] == sb["has_uint32"]
            and sa["uinteger"] == sb["uinteger"])


def test_evolve_matches_reference_goldens(golden, golden_meta):
    for j, ev in enumerate(golden_meta["evolve"]):
        g = I.philox(*ev["pop_key"])
        pop = g.random((ev["N"], ev["G"]))
        fit = g.random(ev["N"])
        if ev["tie"]:
            fit = np.round(fit * 7.0)
        rng = I.philox(*ev["rng_key"])
        params = B.BrkgaParams(population=ev["N"], elite_fraction=ev["elite"],
                               mutant_fraction=ev["mutant"], elite_bias=ev["bias"])
        out = B.evolve(pop, fit, params, rng)
        np.testing.assert_array_equal(out, golden[f"evolve/{j}/out"])
        st = rng.bit_generator.state
        assert [int(x) for x in st["state"]["counter"]] == ev["final_counter"]
        assert int(st["buffer_pos"]) == ev["final_buffer_pos"]
        assert int(st["has_uint32"]) == ev["final_has_uint32"]
        assert int(st["uinteger"]) == ev["final_uinteger"]


@pytest.mark.parametrize("N,G,gens", [(30000, 6, 60), (4097, 33, 40), (25, 9, 50)])
def test_evolve_chain_vs_oracle_including_lemire_rejections(N, G, gens):
    """Many generations: rejections in integers() happen (p ~ 1e-5 per draw at
    N = 30000) and must shift the stream exactly like numpy."""
    params = B.BrkgaParams(population=N)
    host_rng, dev_rng = I.philox(3, N), I.philox(3, N)
    g = I.philox(4, N)
    pop = g.random((N, G))
    dpop = torch.from_numpy(pop).cuda()
    for it in range(gens):
        fit = np.floor(g.random(N) * 50.0)  # many ties
        pop = O.evolve(pop, fit, params.elite_fraction, params.mutant_fraction,
                       params.elite_bias, host_rng)
        dpop = B.evolve(dpop, torch.from_numpy(fit).cuda(), params, dev_rng)
        assert np.array_equal(dpop.cpu().numpy(), pop), f"generation {it}"
        assert same_state(dev_rng, host_rng), f"generator state after generation {it}"


def test_evolve_population_too_small():
    with pytest.raises(B.PopulationTooSmall):
        B.evolve(np.zeros((4, 6)), np.arange(4.0), B.BrkgaParams(population=4), I.philox(0, 0))


def test_evolve_degenerate_bias_copies_elite():  # test_brkga.py:100-107
    pop = np.random.default_rng(3).random((10, 6))
    out = B.evolve(pop, np.arange(10.0), B.BrkgaParams(population=10, elite_bias=1.0),
                   I.philox(3, 3))
    for child in out[2:]:
        assert np.array_equal(child, pop[0])


def test_run_brkga_matches_reference_loop(golden, golden_meta):
    for j, run in enumerate(golden_meta["brkga_runs"]):
        inst = config_instance(run["key"])
        params = B.BrkgaParams(population=run["population"], generations=run["generations"])
        warm = golden[f"brkga/{j}/warm"] if run["warm"] else None
        best, stats = B.run_brkga(inst, params, warm_population=warm, seed=run["seed"])
        np.testing.assert_array_equal([f for _, f in stats.trace], golden[f"brkga/{j}/trace"])
        ops, lens = best.to_arrays(inst.n)
        np.testing.assert_array_equal(ops, golden[f"brkga/{j}/ops"])
        np.testing.assert_array_equal(lens, golden[f"brkga/{j}/lens"])
        assert stats.best_fitness == run["best_fitness"]
        assert stats.decodes == run["decodes"]


def test_decode_single_matches_reference(golden):  # brkga.decode API, batch of one
    inst = config_instance("eil51")
    genes = I.chromosomes(inst.n, 3, (136, 2))
    for i in range(3):
        r = B.decode(genes[i], inst, B.BrkgaParams(population=20))
        assert r.fitness == golden["eil51/dec_fitness"][i]
        assert r.op_visits == golden["eil51/dec_visits"][i]
        ops, lens = r.solution.to_arrays(inst.n)
        np.testing.assert_array_equal(ops, golden["eil51/dec_ops"][i])


def test_run_brkga_monotone_trace_large():
    inst = config_instance("a280")
    params = B.BrkgaParams(population=2000, generations=5)
    best, stats = B.run_brkga(inst, params, seed=1)
    values = [f for _, f in stats.trace]
    assert all(a >= b for a, b in zip(values, values[1:]))
    from paper_2602_23685_b200.schedule import exact_makespan
    assert exact_makespan(inst, best) == stats.best_fitness


@pytest.mark.parametrize("key", [(77, 9), (77, 13), (77, 47)])
def test_evolve_forced_lemire_rejection(key):
    """Philox keys found (by a numpy search over the raw stream) to make numpy
    reject an e_idx (key 9) or o_idx (13, 47) draw in the first generation at
    N = 30000, G = 6: exercises the sequential fix-up path."""
    N, G = 30000, 6
    params = B.BrkgaParams(population=N)
    g = I.philox(5, 5)
    pop = g.random((N, G))
    fit = g.random(N)
    host_rng, dev_rng = I.philox(*key), I.philox(*key)
    ref = O.evolve(pop, fit, params.elite_fraction, params.mutant_fraction, params.elite_bias,
                   host_rng)
    out = B.evolve(pop, fit, params, dev_rng)
    np.testing.assert_array_equal(out, ref)
    assert same_state(dev_rng, host_rng)


def test_single_island_equals_run_brkga():
    """world size 1: the island loop with the device engine is run_brkga."""
    from paper_2602_23685_b200 import islands as IS
    inst = config_instance("eil51")
    params = B.BrkgaParams(population=300, generations=7)
    genes, st = IS.run_islands(inst, params, IS.IslandParams(), seed=4)
    best, stats = B.run_brkga(inst, params, seed=4)
    assert st.global_best == stats.best_fitness
    res = IS.islands_solution(inst, params, genes)
    assert res.solution == best


@pytest.mark.parametrize("skip", [0, 1, 3, 5])
def test_random_device_matches_numpy(skip):
    """vrp_random_fill == Generator(Philox).random, from any buffer position
    and with a pending u32 half (untouched by random())."""
    from paper_2602_23685_b200 import rng as R
    g1 = np.random.Generator(np.random.Philox(key=(31, 7)))
    g2 = np.random.Generator(np.random.Philox(key=(31, 7)))
    for g in (g1, g2):
        g.random(skip)
        g.integers(0, 1000)  # leaves a pending u32 half
    for shape in ((3,), (17, 5), (1000, 3)):
        a = R.random_device(g1, shape).cpu().numpy()
        b = g2.random(shape)
        np.testing.assert_array_equal(a, b)
        assert np.array_equal(R.state_bytes(g1), R.state_bytes(g2))


def test_warm_start_population_device_matches_host():
    from paper_2602_23685_b200 import alns as A
    inst = config_instance("eil51")
    inc = A.construct_initial(inst)
    prm = B.BrkgaParams(population=300, generations=1)
    g1 = np.random.Generator(np.random.Philox(key=(5, 5)))
    g2 = np.random.Generator(np.random.Philox(key=(5, 5)))
    a = B.warm_start_population_device(inst, inc, prm, g1).cpu().numpy()
    b = B.warm_start_population(inst, inc, prm, g2)
    np.testing.assert_array_equal(a, b)
    from paper_2602_23685_b200 import rng as R
    assert np.array_equal(R.state_bytes(g1), R.state_bytes(g2))
