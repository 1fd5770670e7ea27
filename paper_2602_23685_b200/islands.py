"""Multi-GPU BRKGA islands (the reference has no island model,
SPEC.md:457 -- this is new behaviour, parity is per island).

One process per GPU (``torch.distributed``, NCCL over NVLink/NVSwitch).  The
population is split across ranks; each rank runs its own island -- the
device-resident generation step of ``brkga.run_brkga`` (K4 evolve -> K3
decode -> best tracking) with its own Philox stream
``(seed, BRKGA_STREAM + rank)``.  Two exchanges, both tiny next to a
generation:

* **elite migration** every ``migration_interval`` generations: each island
  sends its ``migrants`` best chromosomes (stable fitness order) to rank
  ``(r + 1) % W`` and receives its predecessor's, which replace its worst
  rows (ring ``isend``/``irecv``; k x 4n x 8 B, 1 MB at k = 32, n = 999).
* **incumbent** every ``sync_interval`` generations and at the end: a
  min-all-reduce of the best fitness, then a min-all-reduce of
  ``rank if mine == min else W`` for a deterministic winner (lowest rank on
  ties), then a broadcast of the winner's chromosome.

The collective code is written against an engine interface (``IslandEngine``)
so it is exercised by world-size-2 gloo tests on CPU with a test-only
engine; ``DeviceIslandEngine`` is the product engine.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import brkga as B
from . import rng as R


@dataclass
class IslandParams:
    migration_interval: int = 10
    migrants: int = 32
    sync_interval: int = 10

    def __post_init__(self):
        if self.migration_interval < 1 or self.sync_interval < 1 or self.migrants < 0:
            raise ValueError("intervals must be >= 1 and migrants >= 0")


@dataclass
class IslandStats:
    generations: int = 0
    migrations: int = 0
    syncs: int = 0
    island_best: float = math.inf
    global_best: float = math.inf
    winner: int = -1
    trace: list = field(default_factory=list)  # (generation, global best) at each sync


class IslandEngine:
    """What the island loop needs from a BRKGA implementation.

    pop [N, G] fp64 and fit [N] fp64 tensors on ``device``; best_fit/best_genes
    the island incumbent."""
    device: torch.device
    pop: torch.Tensor
    fit: torch.Tensor
    best_fit: torch.Tensor
    best_genes: torch.Tensor

    def generation(self) -> None:  # evolve + decode non-elites + best update
        raise NotImplementedError

    def order(self) -> torch.Tensor:  # stable fitness order (int64 indices)
        raise NotImplementedError

    def admit(self, rows: torch.Tensor, genes: torch.Tensor, fits: torch.Tensor) -> None:
        """Overwrite population rows with immigrants (and consider them for the incumbent)."""
        self.pop[rows] = genes
        self.fit[rows] = fits
        j = int(torch.argmin(fits).item())
        if fits[j] < self.best_fit[0]:
            self.best_fit[0] = fits[j]
            self.best_genes.copy_(genes[j])


class DeviceIslandEngine(IslandEngine):
    """The island on the local GPU, through the C-ABI (K3 decode, K4 evolve)."""

    def __init__(self, instance, params: B.BrkgaParams, population: np.ndarray, gen, stream=None):
        from . import _native as N
        self.N = N
        self.instance, self.params, self.stream = instance, params, stream
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.pop = torch.from_numpy(np.ascontiguousarray(population)).to(self.device)
        self.size, self.G = self.pop.shape
        self.pop2 = torch.empty_like(self.pop)
        self.fit = torch.empty(self.size, dtype=torch.float64, device=self.device)
        self.fit2 = torch.empty_like(self.fit)
        self.state = R.state_to_device(gen, self.device)
        self.gen = gen
        self.n_elite = int(params.elite_fraction * self.size)
        self.ord = torch.empty(self.size, dtype=torch.int32, device=self.device)
        self.elite_fit = torch.empty(max(self.n_elite, 1), dtype=torch.float64, device=self.device)
        self.best_fit = torch.full((1,), math.inf, dtype=torch.float64, device=self.device)
        self.best_idx = torch.full((1,), -1, dtype=torch.int64, device=self.device)
        self.best_genes = torch.zeros(self.G, dtype=torch.float64, device=self.device)
        self._decode(self.pop, self.fit)
        self._best(self.fit, 0, self.pop)

    def _decode(self, genes, fit_out):
        scratch = {"fitness": fit_out, "makespan": torch.empty_like(fit_out),
                   "scheduled": torch.empty(fit_out.shape, dtype=torch.int32, device=self.device),
                   "visits": torch.empty(fit_out.shape, dtype=torch.int64, device=self.device)}
        B.decode_population(self.instance, genes, self.params, want_solution=False,
                            stream=self.stream, out=scratch)

    def _best(self, fit, lo, genes):
        N = self.N
        N.check(N.lib().vrp_best_update(N.ptr(fit), lo, self.size, N.ptr(genes), self.G,
                                        N.ptr(self.best_fit), N.ptr(self.best_genes),
                                        N.ptr(self.best_idx), None, N.stream_handle(self.stream)),
                "vrp_best_update")

    def generation(self):
        B.evolve_device(self.pop, self.fit, self.params, self.state, out=self.pop2, order=self.ord,
                        elite_fit=self.elite_fit, stream=self.stream)
        self.fit2[:self.n_elite].copy_(self.elite_fit[:self.n_elite])
        self._decode(self.pop2[self.n_elite:], self.fit2[self.n_elite:])
        self._best(self.fit2, self.n_elite, self.pop2)
        self.pop, self.pop2 = self.pop2, self.pop
        self.fit, self.fit2 = self.fit2, self.fit

    def order(self):
        N = self.N
        N.check(N.lib().vrp_fitness_order(N.ptr(self.fit), self.size, N.ptr(self.ord),
                                          N.stream_handle(self.stream)), "vrp_fitness_order")
        return self.ord.to(torch.int64)

    def finish(self):
        R.state_from_device(self.gen, self.state)


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _host_staged(group) -> bool:
    """gloo has no CUDA point-to-point path: stage device tensors through the
    host (the NCCL path sends device memory directly over NVLink)."""
    return dist.get_backend(group) == "gloo"


def _wire(t: torch.Tensor, staged: bool) -> torch.Tensor:
    return t.cpu() if staged and t.is_cuda else t


def migrate(engine: IslandEngine, k: int, group=None) -> None:
    """Ring migration: my k best -> rank+1; rank-1's k best replace my k worst."""
    rank, world = _world(group)
    if world < 2 or k < 1:
        return
    order = engine.order()
    k = min(k, engine.pop.shape[0] // 2)
    staged = _host_staged(group)
    send_genes = _wire(engine.pop[order[:k]].contiguous(), staged)
    send_fit = _wire(engine.fit[order[:k]].contiguous(), staged)
    recv_genes = torch.empty_like(send_genes)
    recv_fit = torch.empty_like(send_fit)
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    ops = [dist.P2POp(dist.isend, send_genes, nxt, group), dist.P2POp(dist.isend, send_fit, nxt, group),
           dist.P2POp(dist.irecv, recv_genes, prv, group), dist.P2POp(dist.irecv, recv_fit, prv, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    worst = order[-k:]
    dev = engine.pop.device
    engine.admit(worst, recv_genes.to(dev), recv_fit.to(dev))


def sync_incumbent(engine: IslandEngine, group=None):
    """Global best over islands: min-all-reduce of the fitness, deterministic
    winner (lowest rank among equals), broadcast of its chromosome.
    Returns (global best fitness, winner rank, chromosome tensor)."""
    rank, world = _world(group)
    best = engine.best_fit.clone()
    genes = engine.best_genes.clone()
    if world < 2:
        return float(best.item()), 0, genes
    dev = genes.device
    staged = _host_staged(group)
    best, genes = _wire(best, staged), _wire(genes, staged)
    gmin = best.clone()
    dist.all_reduce(gmin, op=dist.ReduceOp.MIN, group=group)
    cand = torch.tensor([rank if bool(best.item() == gmin.item()) else world],
                        dtype=torch.int64, device=best.device)
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    winner = int(cand.item())
    src = dist.get_global_rank(group, winner) if group is not None else winner
    dist.broadcast(genes, src=src, group=group)
    return float(gmin.item()), winner, genes.to(dev)


def run_islands(instance, params: B.BrkgaParams, island: IslandParams | None = None, seed: int = 0,
                warm_population=None, group=None, engine_factory=None):
    """BRKGA island model: params.population is the GLOBAL population, split
    evenly over the ranks of ``group``.  Returns (best Solution, IslandStats);
    every rank returns the same global best."""
    island = island or IslandParams()
    rank, world = _world(group)
    size = max(2, params.population // world)
    gen = R.philox_generator(seed, R.BRKGA_STREAM + rank)
    if warm_population is not None:
        pop = np.array(warm_population, dtype=float)[rank * size:(rank + 1) * size]
        if pop.shape[0] < size:
            pop = np.concatenate([pop, gen.random((size - pop.shape[0], 4 * instance.n))])
    else:
        pop = gen.random((size, 4 * instance.n))
    local = B.BrkgaParams(**{**params.__dict__, "population": size})
    make = engine_factory or (lambda inst, prm, p, g: DeviceIslandEngine(inst, prm, p, g))
    engine = make(instance, local, pop, gen)
    stats = IslandStats()
    for g in range(1, params.generations + 1):
        engine.generation()
        if world > 1 and g % island.migration_interval == 0:
            migrate(engine, island.migrants, group)
            stats.migrations += 1
        if g % island.sync_interval == 0:
            best, _, _ = sync_incumbent(engine, group)
            stats.syncs += 1
            stats.trace.append((g, best))
    best, winner, genes = sync_incumbent(engine, group)
    if hasattr(engine, "finish"):
        engine.finish()
    stats.generations = params.generations
    stats.island_best = float(engine.best_fit.item())
    stats.global_best = best
    stats.winner = winner
    return genes, stats


def islands_solution(instance, params: B.BrkgaParams, genes: torch.Tensor):
    """Decode the broadcast winner chromosome into a Solution (device)."""
    res = B.decode_population(instance, genes.view(1, -1), params)
    return B._result(res, 0)
