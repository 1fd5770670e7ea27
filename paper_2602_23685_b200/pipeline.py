"""ALNS -> warm-started BRKGA pipeline -- the reference's
``vrp_rpd.bench.run_pipeline`` (``pkg/src/vrp_rpd/bench.py:204-222``), the
one orchestration entry point on the hot path.  Every stage
runs on the GPU (alns.py, brkga.py); the reference's PCG64 streams become
Philox streams (rng.py) -- the warm-start generator included, so the
pipeline equals the reference's with that single substitution.
"""
from __future__ import annotations

import time

from . import alns as A
from . import brkga as B
from . import rng as R
from .schedule import Solution, evaluate


def run_pipeline(instance, alns_params: A.AlnsParams, brkga_params: B.BrkgaParams, seed: int,
                 pool_size: int = 1, incumbent: Solution | None = None):
    """Returns (better of the two stages, ALNS incumbent)."""
    if incumbent is None:
        if pool_size > 1:
            incumbent, _ = A.run_pool(instance, alns_params, pool_size, seed)
        else:
            incumbent, _ = A.run_alns(instance, alns_params, seed)
    rng = R.philox_generator(A.worker_seed(seed, 7001), R.BRKGA_STREAM)
    warm = B.warm_start_population(instance, incumbent, brkga_params, rng)
    refined, _ = B.run_brkga(instance, brkga_params, warm_population=warm,
                             seed=A.worker_seed(seed, 7002))
    z_inc = evaluate(instance, incumbent).makespan
    z_ref = evaluate(instance, refined).makespan
    return (refined if z_ref <= z_inc else incumbent), incumbent


def run_pipeline_budget(instance, seconds: float, alns_share: float = 0.5, pool_size: int = 32,
                        alns_params: A.AlnsParams | None = None,
                        brkga_params: B.BrkgaParams | None = None, seed: int = 0,
                        initial: Solution | None = None):
    """Best makespan found within a wall-clock budget (the BASELINE metric's
    'best makespan at fixed time'): device-resident ALNS workers (one warp
    each, vrp_alns_iterate) for ``alns_share`` of the budget, then BRKGA generations
    warm-started from the ALNS incumbent for the rest.  Returns
    (best Solution, best makespan, trace [(seconds, best)])."""
    t0 = time.perf_counter()
    alns_params = alns_params or A.AlnsParams(max_iter=200_000)
    brkga_params = brkga_params or B.BrkgaParams(population=4096, generations=1)
    trace = []
    init = initial if initial is not None else A.construct_initial(instance, seed)
    workers = [A._Worker(instance, alns_params, A.worker_seed(seed, i), init, None, None, i)
               for i in range(pool_size)]
    best = min(((w.z_best, w.best) for w in workers), key=lambda x: x[0])
    trace.append((time.perf_counter() - t0, best[0]))

    def stop():
        nonlocal best
        w = min(workers, key=lambda w: w.z_best)
        if w.z_best < best[0]:
            best = (w.z_best, w.best)
            trace.append((time.perf_counter() - t0, best[0]))
        return time.perf_counter() - t0 >= alns_share * seconds

    if alns_params.max_iter:
        A._DeviceWorkers(instance, alns_params, workers).drive(stop=stop, max_stretch=25)
    incumbent = best[1]
    rng = R.philox_generator(A.worker_seed(seed, 7001), R.BRKGA_STREAM)
    pop = B.warm_start_population(instance, incumbent, brkga_params, rng)
    gen = 0
    while time.perf_counter() - t0 < seconds:
        gen += 1
        sol, stats = B.run_brkga(instance, brkga_params, warm_population=pop,
                                 seed=A.worker_seed(seed, 7002 + gen))
        z = evaluate(instance, sol).makespan
        if z < best[0]:
            best = (z, sol)
            trace.append((time.perf_counter() - t0, z))
        pop = B.warm_start_population(instance, best[1], brkga_params, rng)
    return best[1], best[0], trace
