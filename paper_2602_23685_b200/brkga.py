"""BRKGA with the multi-pass decoder -- drop-in for the reference's
``vrp_rpd.brkga`` (``/root/reference/pkg/src/vrp_rpd/brkga.py``).

Device path (C-ABI, csrc/decode.cu + csrc/evolve.cu):
  decode / decode_population   brkga.py:92-207   K3 vrp_decode_batch
  evolve                       brkga.py:231-252  K4 vrp_evolve
  run_brkga                    brkga.py:432-471  device-resident generation loop:
                               K4 evolve -> K3 decode of the non-elite rows ->
                               vrp_best_update, no host round trip per generation
Host (one-off set-up, not on the scoring path; §8(f) row 2):
  encode / perturb / warm-start constructors / warm_start_population
  (brkga.py:210-424), numpy with the reference's draw order.

RNG: ``evolve(..., rng)`` consumes a ``Generator(Philox)`` exactly as numpy
would (bit-identical populations and final generator state).  ``run_brkga``
seeds ``Generator(Philox(key=(seed, BRKGA_STREAM)))`` where the reference
seeds PCG64 (see rng.py); pass ``rng=`` to drive it with your own Philox
generator.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import device as Dev
from . import rng as R
from .schedule import OpKind, Solution

_D, _P = OpKind.DROPOFF, OpKind.PICKUP
_GENE_MAX = np.nextafter(1.0, 0.0)
WARM_SEED_COUNT = 20


class PopulationTooSmall(Exception):
    """Elite or non-elite pool would be empty at this population size."""


@dataclass
class BrkgaParams:
    population: int = 30000
    elite_fraction: float = 0.15
    mutant_fraction: float = 0.15
    elite_bias: float = 0.7
    generations: int = 20000
    warm_start_fraction: float = 0.15
    infeasibility_penalty: float = 1e6
    wait_relaxation: bool = True

    def __post_init__(self):
        if self.elite_fraction + self.mutant_fraction >= 1.0:
            raise ValueError("elite and mutant fractions must sum below 1")
        if not 0.5 < self.elite_bias <= 1.0:
            raise ValueError("elite bias must lie in (0.5, 1]")


@dataclass
class DecodedResult:
    solution: Solution
    fitness: float
    scheduled_count: int
    makespan: float
    op_visits: int


@dataclass
class BrkgaStats:
    generations: int = 0
    decodes: int = 0
    best_fitness: float = math.inf
    trace: list = field(default_factory=list)


def op_index(customer: int, kind: OpKind) -> int:
    return 2 * (customer - 1) + (kind is _P)


def random_population(n: int, size: int, rng) -> np.ndarray:
    return rng.random((size, 4 * n))


def _hint_vehicle(m: int, gene: float) -> int:
    """floor(m*gene) guarded against a float ulp below the next bucket."""
    x = m * gene
    h = int(x)
    if x - h > 1.0 - 1e-9:
        h += 1
    return min(h, m - 1)


# --------------------------------------------------------------------------
# decode (device)
# --------------------------------------------------------------------------

def decode_population(instance, genes, params: BrkgaParams | None = None, want_solution=True,
                      op_dtype=torch.int32, stream=None, out=None):
    """K3 over rows of ``genes`` ([N, 4n] fp64, numpy or torch); device tensors out."""
    params = params or BrkgaParams(population=2)
    return Dev.decode_batch(instance, genes, relax=params.wait_relaxation,
                            penalty=params.infeasibility_penalty, want_solution=want_solution,
                            op_dtype=op_dtype, stream=stream, out=out)


def _result(res, i: int) -> DecodedResult:
    ops = res["ops"][i].cpu().numpy()
    lens = res["lens"][i].cpu().numpy()
    return DecodedResult(solution=Solution.from_arrays(ops, lens),
                         fitness=float(res["fitness"][i].item()),
                         scheduled_count=int(res["scheduled"][i].item()),
                         makespan=float(res["makespan"][i].item()),
                         op_visits=int(res["visits"][i].item()))


def decode(chromosome, instance, params: BrkgaParams) -> DecodedResult:
    genes = np.ascontiguousarray(chromosome, dtype=np.float64).reshape(1, -1)
    return _result(decode_population(instance, genes, params), 0)


# --------------------------------------------------------------------------
# encode / perturb (host)
# --------------------------------------------------------------------------

def encode(instance, solution: Solution) -> np.ndarray:
    """priority (r-1)/L_v at 1-based route position r, hint v/m (brkga.py:210-222)."""
    n, m = instance.n, instance.m
    genes = np.zeros(4 * n)
    for v, tour in enumerate(solution.tours):
        length = len(tour)
        for r, (c, kind) in enumerate(tour):
            o = op_index(c, kind)
            genes[o] = r / length
            genes[2 * n + o] = v / m
    return genes


def perturb(chromosome, rng) -> np.ndarray:
    noise = rng.uniform(-0.03, 0.03, size=len(chromosome))
    return np.clip(chromosome + noise, 0.0, _GENE_MAX)


# --------------------------------------------------------------------------
# evolve (device)
# --------------------------------------------------------------------------

def evolve_device(pop: torch.Tensor, fit: torch.Tensor, params: BrkgaParams, state: torch.Tensor,
                  out: torch.Tensor | None = None, order: torch.Tensor | None = None,
                  elite_fit: torch.Tensor | None = None, stream=None):
    """K4 on device tensors; ``state`` is the 96-byte device generator state."""
    size, genes = pop.shape
    out = out if out is not None else torch.empty_like(pop)
    order = order if order is not None else torch.empty(size, dtype=torch.int32, device=pop.device)
    rc = N.lib().vrp_evolve(N.ptr(pop), N.ptr(fit), size, genes, float(params.elite_fraction),
                            float(params.mutant_fraction), float(params.elite_bias), N.ptr(state),
                            N.ptr(out), N.ptr(order), N.ptr(elite_fit), N.stream_handle(stream))
    if rc == N.VRP_EINVAL and b"PopulationTooSmall" in N.lib(False).vrp_last_error():
        raise PopulationTooSmall(f"population {size} cannot sustain elites")
    N.check(rc, "vrp_evolve")
    return out, order


def evolve(population, fitnesses, params: BrkgaParams, rng):
    """One generation (brkga.py:231-252) on the GPU.  Returns the same type as
    ``population`` (numpy in -> numpy out).  ``rng`` is advanced exactly as
    the reference advances it when it is a Generator(Philox)."""
    size = np.shape(population)[0]
    n_elite = int(params.elite_fraction * size)
    if n_elite < 1 or size - n_elite < 1:
        raise PopulationTooSmall(f"population {size} cannot sustain elites")
    gen = R.as_philox(rng)
    as_numpy = not isinstance(population, torch.Tensor)
    pop = Dev._cuda(population, torch.float64)
    fit = Dev._cuda(fitnesses, torch.float64)
    state = R.state_to_device(gen, pop.device)
    out, _ = evolve_device(pop, fit, params, state)
    R.state_from_device(gen, state)
    return out.cpu().numpy() if as_numpy else out


# --------------------------------------------------------------------------
# warm start (host, one-off)
# --------------------------------------------------------------------------

def _arrays(instance):
    d, p = instance.arrays() if hasattr(instance, "arrays") else (
        np.asarray(instance.d, np.float64), np.asarray(instance.p, np.float64))
    return d, p


def _greedy_ops_solution(instance) -> Solution:
    """Earliest-completion (op, vehicle) pair first, ties by (pickup?, c, v)
    (brkga.py:260-297)."""
    n, m, k = instance.n, instance.m, instance.k
    d, p = _arrays(instance)
    t = np.zeros(m)
    q = [k] * m
    loc = [0] * m
    tours = [[] for _ in range(m)]
    undropped = np.ones(n + 1, bool)
    undropped[0] = False
    ready = np.full(n + 1, np.nan)  # pickup-ready time of dropped, unpicked customers
    left = 2 * n
    while left:
        best = None
        drop_c = np.flatnonzero(undropped)
        pick_c = np.flatnonzero(~np.isnan(ready))
        for v in range(m):
            if q[v] > 0 and drop_c.size:
                comp = t[v] + d[loc[v], drop_c]
                j = int(np.argmin(comp))
                key = (comp[j], 0, int(drop_c[j]), v)
                best = key if best is None or key < best else best
            if q[v] < k and pick_c.size:
                arr = t[v] + d[loc[v], pick_c]
                rdy = ready[pick_c]
                comp = np.where(arr >= rdy, arr, rdy)
                j = int(np.argmin(comp))
                key = (comp[j], 1, int(pick_c[j]), v)
                best = key if best is None or key < best else best
        comp, is_pick, c, v = best
        t[v] = comp
        loc[v] = c
        if is_pick:
            q[v] += 1
            ready[c] = np.nan
            tours[v].append((c, _P))
        else:
            q[v] -= 1
            undropped[c] = False
            ready[c] = comp + p[c]
            tours[v].append((c, _D))
        left -= 1
    return Solution.from_lists(tours)


def _route_group(instance, customers) -> list:
    """Single-vehicle nearest-feasible-operation route (brkga.py:314-347)."""
    d, p = _arrays(instance)
    k = instance.k
    tour = []
    t, loc, q = 0.0, 0, k
    todo = sorted(customers)
    waiting: dict = {}
    while todo or waiting:
        best = None
        if q > 0:
            for c in todo:
                key = (d[loc, c], 0, c)
                if best is None or key < best:
                    best = key
        if q < k:
            for c, rdy in waiting.items():
                arr = t + d[loc, c]
                key = ((arr if arr >= rdy else rdy) - t, 1, c)
                if best is None or key < best:
                    best = key
        _, is_pick, c = best
        if is_pick:
            arr = t + d[loc, c]
            rdy = waiting.pop(c)
            t = arr if arr >= rdy else rdy
            q += 1
            tour.append((c, _P))
        else:
            t += d[loc, c]
            todo.remove(c)
            waiting[c] = t + p[c]
            q -= 1
            tour.append((c, _D))
        loc = c
    return tour


def _load_balanced_solution(instance) -> Solution:
    """Heaviest customer (2 d(0,c) + p_c) onto the lightest vehicle, then route
    each group (brkga.py:300-311)."""
    d, p = _arrays(instance)
    m = instance.m
    w = {c: 2.0 * d[0, c] + p[c] for c in instance.customers}
    load = [0.0] * m
    groups = [[] for _ in range(m)]
    for c in sorted(instance.customers, key=lambda c: (-w[c], c)):
        v = min(range(m), key=lambda u: (load[u], u))
        groups[v].append(c)
        load[v] += w[c]
    return Solution.from_lists([_route_group(instance, g) for g in groups])


def _spt_solution(instance) -> Solution:
    """Dropoffs by ascending processing time, each to the earliest-arriving
    vehicle (any vehicle -- the reference's quirk); the cheapest
    ready pickup is taken whenever every vehicle is empty (brkga.py:350-391)."""
    d, p = _arrays(instance)
    m, k = instance.m, instance.k
    t = [0.0] * m
    q = [k] * m
    loc = [0] * m
    tours = [[] for _ in range(m)]
    waiting: dict = {}

    def take_pickup():
        best = None
        for v in range(m):
            if q[v] >= k:
                continue
            for c, rdy in waiting.items():
                arr = t[v] + d[loc[v], c]
                key = (arr if arr >= rdy else rdy, c, v)
                if best is None or key < best:
                    best = key
        comp, c, v = best
        t[v] = comp
        loc[v] = c
        q[v] += 1
        del waiting[c]
        tours[v].append((c, _P))

    for c in sorted(instance.customers, key=lambda c: (p[c], c)):
        while all(x <= 0 for x in q):
            take_pickup()
        v = min(range(m), key=lambda u: (t[u] + d[loc[u], c], u))
        t[v] += d[loc[v], c]
        loc[v] = c
        q[v] -= 1
        waiting[c] = t[v] + p[c]
        tours[v].append((c, _D))
    while waiting:
        take_pickup()
    return Solution.from_lists(tours)


def warm_start_seeds(instance, incumbent: Solution) -> list:
    return [encode(instance, incumbent), encode(instance, _greedy_ops_solution(instance)),
            encode(instance, _load_balanced_solution(instance)),
            encode(instance, _spt_solution(instance))]


def warm_start_population_device(instance, alns_solution: Solution, params: BrkgaParams, rng) -> torch.Tensor:
    """warm_start_population with the uniform fill drawn on the device
    (vrp_random_fill); identical values and generator state, as a device
    tensor for run_brkga."""
    n_p = params.population
    seeds = warm_start_seeds(instance, alns_solution)
    while len(seeds) < WARM_SEED_COUNT:
        seeds.append(perturb(seeds[0], rng))
    n_warm = min(n_p, math.ceil(params.warm_start_fraction * n_p))
    pop = R.random_device(rng, (n_p, 4 * instance.n))
    rows = [seeds[slot] if slot < len(seeds) else perturb(seeds[slot % len(seeds)], rng)
            for slot in range(n_warm)]
    if rows:
        pop[:n_warm] = torch.from_numpy(np.stack(rows)).to(pop.device)
    return pop


def warm_start_population(instance, alns_solution: Solution, params: BrkgaParams, rng) -> np.ndarray:
    """ceil(warm_start_fraction * N_p) warm slots cycling through 20 seeds
    (brkga.py:405-424), same draw order as the reference."""
    n_p = params.population
    seeds = warm_start_seeds(instance, alns_solution)
    while len(seeds) < WARM_SEED_COUNT:
        seeds.append(perturb(seeds[0], rng))
    n_warm = min(n_p, math.ceil(params.warm_start_fraction * n_p))
    pop = rng.random((n_p, 4 * instance.n))
    for slot in range(n_warm):
        pop[slot] = seeds[slot] if slot < len(seeds) else perturb(seeds[slot % len(seeds)], rng)
    return pop


# --------------------------------------------------------------------------
# main loop (device resident)
# --------------------------------------------------------------------------

def run_brkga(instance, params: BrkgaParams, warm_population=None, seed: int = 0, rng=None,
              stream=None, deadline: float | None = None):
    """Evolve for params.generations generations entirely on the GPU; returns
    (best Solution, BrkgaStats) like brkga.py:432-471.  ``deadline``
    (time.perf_counter() value, not in the reference) stops early at a
    generation boundary -- the time-budgeted pipeline uses it."""
    gen = R.as_philox(rng) if rng is not None else R.philox_generator(seed, R.BRKGA_STREAM)
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(warm_population, torch.Tensor):
        pop = warm_population.to(dev, torch.float64).clone()
    elif warm_population is not None:
        pop = torch.from_numpy(np.array(warm_population, dtype=float, copy=True)).to(dev)
    else:  # rng.random((N_p, 4n)) (brkga.py:436-437), drawn on the device
        pop = R.random_device(gen, (params.population, 4 * instance.n), dev)
    size, G = pop.shape
    pop2 = torch.empty_like(pop)
    fits = torch.empty(size, dtype=torch.float64, device=dev)
    fits2 = torch.empty_like(fits)
    state = R.state_to_device(gen, dev)
    order = torch.empty(size, dtype=torch.int32, device=dev)
    n_elite = int(params.elite_fraction * size)
    elite_fit = torch.empty(max(n_elite, 1), dtype=torch.float64, device=dev)
    best_fit = torch.full((1,), math.inf, dtype=torch.float64, device=dev)
    best_idx = torch.full((1,), -1, dtype=torch.int64, device=dev)
    best_genes = torch.empty(G, dtype=torch.float64, device=dev)
    trace = torch.empty(params.generations + 1, dtype=torch.float64, device=dev)
    L = N.lib()
    sh = N.stream_handle(stream)

    def decode_rows(genes, fit_out):
        scratch = {"fitness": fit_out, "makespan": torch.empty_like(fit_out),
                   "scheduled": torch.empty(fit_out.shape, dtype=torch.int32, device=dev),
                   "visits": torch.empty(fit_out.shape, dtype=torch.int64, device=dev)}
        decode_population(instance, genes, params, want_solution=False, stream=stream, out=scratch)

    def best_update(fit, lo, genes, slot):
        N.check(L.vrp_best_update(N.ptr(fit), lo, size, N.ptr(genes), G, N.ptr(best_fit),
                                  N.ptr(best_genes), N.ptr(best_idx), N.ptr(trace[slot:slot + 1]),
                                  sh), "vrp_best_update")

    decode_rows(pop, fits)
    best_update(fits, 0, pop, 0)
    done = params.generations
    for g in range(1, params.generations + 1):
        if deadline is not None and g % 2 == 1:
            torch.cuda.synchronize()
            if time.perf_counter() >= deadline:
                done = g - 1
                break
        evolve_device(pop, fits, params, state, out=pop2, order=order, elite_fit=elite_fit,
                      stream=stream)
        fits2[:n_elite].copy_(elite_fit[:n_elite])
        decode_rows(pop2[n_elite:], fits2[n_elite:])
        best_update(fits2, n_elite, pop2, g)
        # the incumbent row index refers to this generation's buffer; rows
        # are never compared across buffers, only fitness values
        pop, pop2 = pop2, pop
        fits, fits2 = fits2, fits
    R.state_from_device(gen, state)
    best = _result(decode_population(instance, best_genes.view(1, G), params, stream=stream), 0)
    tr = trace.cpu().tolist()[:done + 1]
    stats = BrkgaStats(generations=done,
                       decodes=size + done * (size - n_elite),
                       best_fitness=best.fitness, trace=list(enumerate(tr)))
    return best.solution, stats
