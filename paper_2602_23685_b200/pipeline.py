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


def run_pipeline_budget(instance, seconds: float, alns_share: float = 0.8, pool_size: int = 296,
                        alns_params: A.AlnsParams | None = None,
                        brkga_params: B.BrkgaParams | None = None, seed: int = 0,
                        initial: Solution | None = None, fit_cooling: bool = True,
                        polish: bool = True, polish_share: float | None = None,
                        final_share: float | None = None,
                        alns_max_n: int = 400, exchange=None, diversify: int = 0):
    """Best makespan found within a wall-clock budget (the BASELINE metric's
    'best makespan at fixed time'; the reference has no budget).

    Stage 0 (``polish``): the device first-improvement polish
    (baselines.two_opt_improve: 2-opt / relocate / swap neighbourhoods scored
    by K1 at tens of millions of candidates per second) takes the
    constructed solution to a local optimum -- capped at ``polish_share`` of
    the budget (default 0.4 for n >= 90; small instances measured better
    when ALNS starts from the constructed solution, so 0 there).
    Stage 1, ``alns_share`` of what remains before the final reserve (only
    for n <= ``alns_max_n``; measured at n = 999, profiles/r02_summary.md:
    the team-repair ALNS runs ~0.5 s per iteration per worker there, but its
    capacity cascades remove 50-200 customers per move and, given the stage,
    it does not improve the polished incumbent -- 299.0 M with the stage vs
    295.7 M without in 60 s -- so the default keeps it for n <= 400):
    ``pool_size`` device-resident ALNS workers (one warp each,
    vrp_alns_iterate) in pools that poll their pool's incumbent.  With
    ``fit_cooling`` the SA schedule is fitted to the stage: a 10-iteration
    calibration stretch measures the iteration rate, and the cooling rate is
    set so that the temperature falls to 1e-3 of its start by the end
    (the reference's alpha = 0.9998 assumes 20,000 iterations).
    Stage 2: one BRKGA run (device generation loop) warm-started from the
    incumbent, stopped at its deadline.
    Stage 3 (``polish``), the last ``final_share`` (0.1 below n = 90, 0.5
    below n = 500, 0.6 above, where BRKGA does not improve on the polished
    solution within a minute):
    standard (restarting) polish of the incumbent, and, if it converges
    before the deadline, iterated local search (random kicks repaired by K5,
    polished) for the rest.
    ``exchange`` (multi-GPU, run_pipeline_budget_distributed): called as
    exchange(z, sol, more) at every stage boundary and after every kick
    round of the tail -- the same number of times on every rank -- it returns
    the global best (z, sol) and whether every rank wants another round.
    Returns (best Solution, best makespan, trace [(seconds, best)])."""
    from . import baselines as BL
    t0 = time.perf_counter()
    end = t0 + seconds
    brkga_params = brkga_params or B.BrkgaParams(population=8192, generations=10**6)
    trace = []
    init = initial if initial is not None else A.construct_initial(instance, seed)
    z0 = evaluate(instance, init).makespan
    best = (z0, init)
    trace.append((time.perf_counter() - t0, z0))
    if diversify:
        # another rank of a multi-GPU run: start the (deterministic) polish from
        # a kicked copy of the construction, so the ranks explore different
        # local optima instead of repeating one
        best = _Kicker(instance, init, seed + 7919 * diversify, q=10).kick()

    def offer(sol):
        nonlocal best
        z = evaluate(instance, sol).makespan
        if z < best[0]:
            best = (z, sol)
            trace.append((time.perf_counter() - t0, z))

    def share(more=True):  # adopt the global incumbent (multi-GPU); returns the ranks' consensus on `more`
        nonlocal best
        if exchange is None:
            return more
        zg, sg, go = exchange(best[0], best[1], more)
        if zg < best[0]:
            best = (zg, sg)
            trace.append((time.perf_counter() - t0, zg))
        return go

    if polish_share is None:
        polish_share = (0.4 if instance.n < 500 else 0.6) if instance.n >= 90 else 0.0
    if final_share is None:  # measured (profiles/r01_summary.md): the polish + kick tail
        final_share = 0.1 if instance.n < 90 else (0.5 if instance.n < 500 else 0.6)
    if polish and polish_share > 0 and time.perf_counter() < end:
        # (restarting scans: at n = 999 they converge in ~25 s to a better optimum
        # than the resumed variant's ~10 s one; below that both take < 1 s)
        offer(BL.two_opt_improve(instance, best[1], move_budget=10**15,
                                 deadline=min(end, t0 + polish_share * seconds)))
    share()
    final_start = end - (final_share * seconds if polish else 0.0)
    now = time.perf_counter()
    alns_end = now + alns_share * max(0.0, final_start - now)
    if instance.n > alns_max_n:
        alns_end = now
    init = best[1]
    per_iter = None
    if alns_params is None and now < alns_end:
        alns_params = A.AlnsParams(max_iter=10)
        if fit_cooling:  # calibration stretch: iteration time of this pool on this instance
            probe = [A._Worker(instance, alns_params, A.worker_seed(seed + 1, i), init, None, None, i)
                     for i in range(pool_size)]
            t1 = time.perf_counter()
            A._DeviceWorkers(instance, alns_params, probe).run(1, 10)
            per_iter = (time.perf_counter() - t1) / 10
            iters = max(50, int((alns_end - time.perf_counter()) / per_iter))
            check = max(25, iters // 20)
            alns_params = A.AlnsParams(max_iter=int(iters * 1.5) + 100,
                                       alpha=min(0.99999, max(0.9, 1e-3 ** (1.0 / iters))),
                                       best_check_interval=check, pool_sync_interval=check)
        else:
            alns_params = A.AlnsParams(max_iter=200_000)
    if alns_params is not None and alns_params.max_iter and time.perf_counter() < alns_end:
        wpp = alns_params.workers_per_pool
        n_pools = (pool_size + wpp - 1) // wpp
        pools = [A._PoolShare() for _ in range(n_pools)]
        gshare = A._PoolShare() if n_pools > 1 else None
        workers = [A._Worker(instance, alns_params, A.worker_seed(seed, i), init,
                             pools[i // wpp] if pool_size > 1 else None, gshare if pool_size > 1 else None, i)
                   for i in range(pool_size)]

        def stop():
            nonlocal best
            w = min(workers, key=lambda w: w.z_best)
            if w.z_best < best[0]:
                best = (w.z_best, w.best)
                trace.append((time.perf_counter() - t0, best[0]))
            return time.perf_counter() >= alns_end

        # stretches of <= ~2 s so that the stage ends near its deadline (an
        # iteration takes ~0.5 s per worker at n = 999)
        stretch = 25 if per_iter is None else max(1, min(25, int(2.0 / max(per_iter, 1e-6))))
        A._DeviceWorkers(instance, alns_params, workers).drive(stop=stop, max_stretch=stretch)
    share()
    if time.perf_counter() < final_start:
        rng = R.philox_generator(A.worker_seed(seed, 7001), R.BRKGA_STREAM)
        pop = B.warm_start_population_device(instance, best[1], brkga_params, rng)
        sol, _ = B.run_brkga(instance, brkga_params, warm_population=pop, seed=A.worker_seed(seed, 7002),
                             deadline=final_start)
        offer(sol)
    share()
    if polish and time.perf_counter() < end:
        offer(BL.two_opt_improve(instance, best[1], move_budget=10**15, deadline=end))
    if polish:
        # time left at a local optimum: iterated local search (batched random
        # kicks -> K5 greedy repair -> K1 -> polish of the best kick); with
        # several GPUs the ranks exchange their incumbent after every round,
        # continue from the global best and stop together
        kick = _Kicker(instance, best[1], seed)
        while share(time.perf_counter() + 1.2 * kick.last_s < end - 0.5):
            sol = kick.round(end)
            if sol is not None:
                offer(sol)
            kick.adopt(best[0], best[1])
    return best[1], best[0], trace


class _Kicker:
    """Iterated local search for the tail of a budget, one round per call:
    destroy ``q`` random customers of the current solution in ``batch``
    independent ways (K6), greedily repair them (K5), score them (K1) and
    polish the best one (resumed first-improvement scans).  ``round`` returns
    the polished solution when it improves on the current one (else None);
    ``adopt`` hands over an external incumbent (another GPU's)."""

    def __init__(self, instance, start: Solution, seed: int, batch: int = 64, q: int = 5):
        import torch
        self.instance, self.batch = instance, batch
        self.rng = R.philox_generator(A.worker_seed(seed, 7100), R.ALNS_STREAM)
        self.cur, self.zcur = start, evaluate(instance, start).makespan
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.q = min(q if instance.n < 500 else 2, instance.n)  # removals cascade; large n: smaller kicks
        self.last_s = 0.0  # duration of the last kick step (repairs do not watch the clock)

    def adopt(self, z: float, sol: Solution) -> None:
        if z < self.zcur:
            self.cur, self.zcur = sol, z

    def kick(self):
        """The best of one batch of kicks of the current solution (no polish):
        (makespan, Solution); the current solution when no kick repairs."""
        sol = self.round(None, polish=False)
        return (evaluate(self.instance, sol).makespan, sol) if sol is not None else (self.zcur, self.cur)

    def round(self, deadline, polish: bool = True):
        import numpy as np
        import torch
        from . import baselines as BL
        from . import device as DV
        from . import insertion as INS
        instance, batch, dev, n = self.instance, self.batch, self.dev, self.instance.n
        tk = time.perf_counter()
        o, l = self.cur.to_arrays(n)
        ops = torch.from_numpy(np.tile(o[:2 * n], (batch, 1))).to(dev)
        lens = torch.from_numpy(np.tile(l, (batch, 1))).to(dev)
        gens = [np.random.Generator(np.random.Philox(key=(int(x), 0xC1C)))
                for x in self.rng.integers(0, 2**62, size=batch)]
        states = torch.from_numpy(np.stack([R.state_bytes(g) for g in gens])).to(dev)
        d = DV.destroy_batch(instance, ops, lens, torch.zeros(batch, dtype=torch.int32, device=dev),
                             torch.full((batch,), self.q, dtype=torch.int32, device=dev),
                             min(A.removal_bounds(n)[0], n), states)
        nr = d["nremoved"].cpu().numpy()
        rem = d["removed"].cpu().numpy()
        ro, rl, st = INS.reinsert_batch(instance, d["ops"], d["lens"], [list(rem[i, :nr[i]]) for i in range(batch)],
                                        [0] * batch, None)
        ok = np.flatnonzero(st == 0)
        self.last_s = time.perf_counter() - tk
        if not ok.size:
            return None
        z = DV.makespan_batch(instance, ro[ok], rl[ok], mode=0)
        zs, ss = z["z"].cpu().numpy(), z["status"].cpu().numpy()
        good = np.flatnonzero(ss == 0)
        if not good.size:
            return None
        k = ok[good[np.argmin(zs[good])]]
        kicked = Solution.from_arrays(ro[k], rl[k])
        self.last_s = time.perf_counter() - tk
        if not polish:
            return kicked
        pol = BL.two_opt_improve(instance, kicked, move_budget=10**15, resume=True, deadline=deadline)
        zp = evaluate(instance, pol).makespan
        if zp < self.zcur:
            self.cur, self.zcur = pol, zp
            return pol
        return None


def run_pipeline_budget_distributed(instance, seconds: float, seed: int = 0, group=None, **kw):
    """run_pipeline_budget on every rank of ``group`` (one GPU each; SURVEY
    §8(e): the pipeline's work shards as independent searches) with
    rank-specific seeds; ranks > 0 polish a kicked copy of the construction
    (different local optima).  The ranks cooperate: at every stage boundary and
    after every kick round of the tail they min-all-reduce the best makespan
    and broadcast the winner's routes (alns.sync_pool_share: lowest rank wins
    ties), and continue from the global best; a final exchange makes the
    result identical on every rank.  Every rank returns (best Solution, best makespan,
    its own trace)."""
    rank, world = A._dist_world(group)

    def exchange(z, sol, more):
        if world < 2:
            return z, sol, more
        import torch
        import torch.distributed as dist
        share = A._PoolShare()
        share.offer(rank, z, sol)
        A.sync_pool_share(instance, share, group)
        dev = (torch.device("cuda", torch.cuda.current_device())
               if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        flag = torch.tensor([1 if more else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        return share.best_z, share.best_sol, bool(flag.item())

    sol, z, trace = run_pipeline_budget(instance, seconds, seed=seed + 1009 * rank, exchange=exchange,
                                        diversify=rank, **kw)
    share = A._PoolShare()
    share.offer(rank, z, sol)
    A.sync_pool_share(instance, share, group)
    return share.best_sol, share.best_z, trace
