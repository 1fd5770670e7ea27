"""World-size-2 gloo tests (CPU) of the island collectives: ring elite
migration and the deterministic incumbent all-reduce, over a test-only island
engine built on the CPU oracle (the product engine is DeviceIslandEngine)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleIslandEngine:
    """Island engine over the oracle's decode/evolve (test infrastructure)."""

    def __init__(self, instance, params, population, gen):
        self.instance, self.params, self.gen = instance, params, gen
        self.device = torch.device("cpu")
        self.pop = torch.from_numpy(np.array(population))
        self.fit = torch.from_numpy(O.decode_batch(instance, population)["fitness"].copy())
        j = int(torch.argmin(self.fit))
        self.best_fit = self.fit[j:j + 1].clone()
        self.best_genes = self.pop[j].clone()
        self.n_elite = int(params.elite_fraction * self.pop.shape[0])

    def generation(self):
        p = self.params
        order = O.stable_argsort(self.fit.numpy())
        elite = self.fit.numpy()[order[:self.n_elite]].copy()
        pop = O.evolve(self.pop.numpy(), self.fit.numpy(), p.elite_fraction, p.mutant_fraction,
                       p.elite_bias, self.gen)
        fit = np.empty(pop.shape[0])
        fit[:self.n_elite] = elite
        fit[self.n_elite:] = O.decode_batch(self.instance, pop[self.n_elite:])["fitness"]
        self.pop, self.fit = torch.from_numpy(pop), torch.from_numpy(fit)
        j = self.n_elite + int(np.argmin(fit[self.n_elite:]))
        if fit[j] < self.best_fit[0]:
            self.best_fit[0] = fit[j]
            self.best_genes = self.pop[j].clone()

    def order(self):
        return torch.from_numpy(O.stable_argsort(self.fit.numpy()))

    def admit(self, rows, genes, fits):
        self.pop[rows] = genes
        self.fit[rows] = fits
        j = int(torch.argmin(fits))
        if fits[j] < self.best_fit[0]:
            self.best_fit[0] = fits[j]
            self.best_genes = genes[j].clone()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _migration_case(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).parent))
    sys.path.insert(0, str(Path(__file__).parent / "golden"))
    from test_islands_gloo import OracleIslandEngine  # noqa
    from paper_2602_23685_b200 import brkga as B
    from paper_2602_23685_b200 import islands as IS
    from paper_2602_23685_b200.configs import config_instance
    inst = config_instance("gr17")
    params = B.BrkgaParams(population=40)
    g = np.random.Generator(np.random.Philox(key=(rank, 1)))
    eng = OracleIslandEngine(inst, params, g.random((40, 4 * inst.n)), g)
    before = eng.pop.clone(), eng.fit.clone()
    order = eng.order()
    IS.migrate(eng, 4, None)
    return {"before_pop": before[0].numpy(), "before_fit": before[1].numpy(),
            "order": order.numpy(), "after_pop": eng.pop.numpy(), "after_fit": eng.fit.numpy()}


def test_ring_migration_world2():
    out = run_world(_migration_case)
    for r in (0, 1):
        src = out[1 - r]  # rank r receives from (r - 1) % 2
        me = out[r]
        best4 = src["order"][:4]
        worst4 = me["order"][-4:]
        np.testing.assert_array_equal(me["after_pop"][worst4], src["before_pop"][best4])
        np.testing.assert_array_equal(me["after_fit"][worst4], src["before_fit"][best4])
        keep = np.setdiff1d(np.arange(40), worst4)
        np.testing.assert_array_equal(me["after_pop"][keep], me["before_pop"][keep])


def _sync_case(rank, world):
    from paper_2602_23685_b200 import islands as IS

    class E:
        pass
    e = E()
    # equal best on both ranks: the lowest rank must win
    e.best_fit = torch.tensor([5.0 if rank == 0 else 5.0], dtype=torch.float64)
    e.best_genes = torch.full((6,), float(rank))
    tie = IS.sync_incumbent(e, None)
    e.best_fit = torch.tensor([7.0 if rank == 0 else 3.0], dtype=torch.float64)
    strict = IS.sync_incumbent(e, None)
    return {"tie": (tie[0], tie[1], tie[2].tolist()), "strict": (strict[0], strict[1], strict[2].tolist())}


def test_incumbent_sync_world2():
    out = run_world(_sync_case)
    for r in (0, 1):
        assert out[r]["tie"] == (5.0, 0, [0.0] * 6)
        assert out[r]["strict"] == (3.0, 1, [1.0] * 6)


def _island_run(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).parent))
    sys.path.insert(0, str(Path(__file__).parent / "golden"))
    from test_islands_gloo import OracleIslandEngine  # noqa
    from paper_2602_23685_b200 import brkga as B
    from paper_2602_23685_b200 import islands as IS
    from paper_2602_23685_b200.configs import config_instance
    inst = config_instance("gr17")
    params = B.BrkgaParams(population=80, generations=12)
    genes, stats = IS.run_islands(inst, params, IS.IslandParams(migration_interval=3, migrants=4,
                                                                sync_interval=4),
                                  seed=21, engine_factory=lambda i, p, pop, g: OracleIslandEngine(i, p, pop, g))
    return {"best": stats.global_best, "winner": stats.winner, "island": stats.island_best,
            "genes": genes.numpy(), "trace": stats.trace, "migrations": stats.migrations}


def test_run_islands_world2_consistent():
    out = run_world(_island_run)
    assert out[0]["best"] == out[1]["best"] == min(out[0]["island"], out[1]["island"])
    assert out[0]["winner"] == out[1]["winner"]
    np.testing.assert_array_equal(out[0]["genes"], out[1]["genes"])
    assert out[0]["trace"] == out[1]["trace"]
    vals = [v for _, v in out[0]["trace"]]
    assert all(a >= b for a, b in zip(vals, vals[1:]))
    assert out[0]["migrations"] == 4
    # the broadcast chromosome decodes to the global best fitness
    from conftest import config_instance
    inst = config_instance("gr17")
    fit = O.decode_batch(inst, out[0]["genes"][None, :])["fitness"][0]
    assert fit == out[0]["best"]
    assert math.isfinite(fit)


def _island_dev_vs_oracle(rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).parent))
    sys.path.insert(0, str(Path(__file__).parent / "golden"))
    torch.cuda.set_device(0)  # both ranks share cuda:0; their kernels never wait on each other
    from test_islands_gloo import OracleIslandEngine  # noqa
    from paper_2602_23685_b200 import brkga as B
    from paper_2602_23685_b200 import islands as IS
    from paper_2602_23685_b200.configs import config_instance
    inst = config_instance("eil51")
    params = B.BrkgaParams(population=120, generations=12)
    out = {}
    for kind in ("device", "oracle"):
        made = []

        def factory(i, p, pop, g, kind=kind):
            e = IS.DeviceIslandEngine(i, p, pop, g) if kind == "device" else OracleIslandEngine(i, p, pop, g)
            made.append(e)
            return e
        genes, stats = IS.run_islands(inst, params, IS.IslandParams(migration_interval=3, migrants=5,
                                                                    sync_interval=4),
                                      seed=33, engine_factory=factory)
        e = made[0]
        out[kind] = {"best": stats.global_best, "winner": stats.winner, "island": stats.island_best,
                     "genes": genes.cpu().numpy(), "trace": stats.trace, "migrations": stats.migrations,
                     "pop": e.pop.cpu().numpy(), "fit": e.fit.cpu().numpy(),
                     "key": e.gen.bit_generator.state["state"]["key"].tolist(),
                     "counter": e.gen.bit_generator.state["state"]["counter"].tolist()}
    return out


@pytest.mark.gpu
def test_device_island_engine_world2_equals_oracle_engine():
    """DeviceIslandEngine (K3/K4 through the C-ABI) at world size 2 -- both
    ranks on cuda:0 over gloo, device tensors staged through the host -- equals
    the oracle engine on the same Philox streams: global best, winner,
    broadcast chromosome, sync trace, and every island's final population
    (which holds the migrated rows) and generator state."""
    out = run_world(_island_dev_vs_oracle)
    for r in (0, 1):
        d, o = out[r]["device"], out[r]["oracle"]
        assert d["best"] == o["best"] and d["winner"] == o["winner"] and d["island"] == o["island"]
        assert d["trace"] == o["trace"] and d["migrations"] == o["migrations"] == 4
        np.testing.assert_array_equal(d["genes"], o["genes"])
        np.testing.assert_array_equal(d["pop"], o["pop"])
        np.testing.assert_array_equal(d["fit"], o["fit"])
    assert out[0]["device"]["best"] == out[1]["device"]["best"]
    for r in (0, 1):
        assert out[r]["device"]["counter"] == out[r]["oracle"]["counter"]
    assert out[0]["device"]["key"] != out[1]["device"]["key"]  # independent island streams
