"""Host-side BRKGA pieces (encode, warm-start constructors, warm_start_population)
against the reference's outputs, and the oracle's evolve+decode composition
against the reference's run_brkga loop (driven by Generator(Philox))."""
import numpy as np
import pytest

import inputs as I
from conftest import CONFIG_KEYS, config_instance
from oracle import oracle as O
from paper_2602_23685_b200 import brkga as B
from paper_2602_23685_b200.schedule import Solution

CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


@pytest.mark.parametrize("key", CONFIG_KEYS)
@pytest.mark.parametrize("tag,fn", [("greedy", B._greedy_ops_solution),
                                    ("lb", B._load_balanced_solution),
                                    ("spt", B._spt_solution)])
def test_warm_start_constructors_match_reference(key, tag, fn, golden):
    inst = config_instance(key)
    sol = fn(inst)
    ops, lens = sol.to_arrays(inst.n)
    np.testing.assert_array_equal(ops, golden[f"{key}/ws_{tag}_ops"])
    np.testing.assert_array_equal(lens, golden[f"{key}/ws_{tag}_lens"])
    np.testing.assert_array_equal(B.encode(inst, sol), golden[f"{key}/ws_{tag}_enc"])


@pytest.mark.parametrize("key", ["gr17", "eil51", "kroA100", "a280"])
def test_warm_start_population_matches_reference(key, golden):
    inst = config_instance(key)
    inc = Solution.from_arrays(golden[f"{key}/dec_ops"][0], golden[f"{key}/dec_lens"][0])
    pop = B.warm_start_population(inst, inc, B.BrkgaParams(population=64, generations=3),
                                  I.philox(13, CID[key]))
    np.testing.assert_array_equal(pop, golden[f"{key}/ws_pop"])


def test_encode_reference_points():  # test_brkga.py:36-41
    from paper_2602_23685_b200.instance import FleetConfig, Instance
    toy = Instance(n=2, d=((0, 10, 12), (10, 0, 5), (12, 5, 0)), p=(0, 20, 20),
                   fleet=FleetConfig(1, 2), label="toy")
    genes = B.encode(toy, Solution.from_lists([[(1, "D"), (2, "D"), (1, "P"), (2, "P")]]))
    assert genes[0] == 0.0 and genes[2] == 0.25
    assert np.all(genes >= 0) and np.all(genes < 1)


def test_perturb_bounds_and_clamp():  # test_brkga.py:62-78
    rng = np.random.default_rng(5)
    genes = np.array([0.0, 0.5, 0.999999, 0.01])
    for _ in range(50):
        out = B.perturb(genes, rng)
        assert np.all(out >= 0.0) and np.all(out < 1.0)

    class Down:
        def uniform(self, lo, hi, size):
            return np.full(size, -0.02)
    assert B.perturb(np.zeros(4), Down())[0] == 0.0


def oracle_run_brkga(inst, run, golden, j):
    """The reference's run_brkga loop (brkga.py:432-471) over the oracle's
    decode/evolve, with Generator(Philox(key=(seed, BRKGA_STREAM)))."""
    params = B.BrkgaParams(population=run["population"], generations=run["generations"])
    rng = I.philox(run["seed"], 0xB4C6A)
    if run["warm"]:
        pop = golden[f"brkga/{j}/warm"].copy()
    else:
        pop = rng.random((params.population, 4 * inst.n))
    size = pop.shape[0]
    dec = O.decode_batch(inst, pop)
    fits = dec["fitness"].copy()
    bi = int(np.argmin(fits))
    best_f, best_row = fits[bi], pop[bi].copy()
    trace = [best_f]
    n_elite = int(params.elite_fraction * size)
    for _ in range(params.generations):
        order = O.stable_argsort(fits)
        elite = fits[order[:n_elite]]
        pop = O.evolve(pop, fits, params.elite_fraction, params.mutant_fraction,
                       params.elite_bias, rng)
        fits = np.empty(size)
        fits[:n_elite] = elite
        fits[n_elite:] = O.decode_batch(inst, pop[n_elite:])["fitness"]
        j2 = n_elite + int(np.argmin(fits[n_elite:]))
        if fits[j2] < best_f:
            best_f, best_row = fits[j2], pop[j2].copy()
        trace.append(best_f)
    return np.array(trace), O.decode_batch(inst, best_row[None, :])


def test_oracle_run_brkga_matches_reference_loop(golden, golden_meta):
    for j, run in enumerate(golden_meta["brkga_runs"]):
        inst = config_instance(run["key"])
        trace, best = oracle_run_brkga(inst, run, golden, j)
        np.testing.assert_array_equal(trace, golden[f"brkga/{j}/trace"])
        np.testing.assert_array_equal(best["ops"][0], golden[f"brkga/{j}/ops"])
        np.testing.assert_array_equal(best["lens"][0], golden[f"brkga/{j}/lens"])
