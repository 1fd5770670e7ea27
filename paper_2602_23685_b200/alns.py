"""ALNS with simulated annealing -- drop-in for the reference's ``vrp_rpd.alns``
(``/root/reference/pkg/src/vrp_rpd/alns.py``).

Where the work goes (engine="device", the default):
  iterations         csrc/alns_step.cu (vrp_alns_iterate): one warp per worker
                     runs roulette, destroy (K6), remove_customers, repair (the
                     K5 core), the exact replay, SA acceptance, cooling, reheat
                     and weight updates for a whole stretch of iterations
  local search       pickup_repositioning / cross_agent_relocation at their
                     cadence, batched over all workers (localsearch.py:
                     device-built neighbourhoods, K2 estimate, K1 verify)
  pool sharing       on the host at the stretch boundaries, in the sequential
                     loop's (iteration, worker) order
engine="host" keeps destroy and acceptance on the host with one batched K5 +
K1 launch per iteration (the cross-check of the device engine).  Both follow
the reference's draw order, so one generator per worker behaves exactly like
the reference's single rng.

RNG: ``run_alns(seed)`` uses ``Generator(Philox(key=(seed, ALNS_STREAM)))``
where the reference uses PCG64(seed) (see rng.py); with that substitution the
trajectory is identical to the reference's (tests/test_gpu_alns.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import insertion
from . import rng as R
from .insertion import InsertionContext, RepairFailed
from .schedule import (OpKind, ScheduleError, Solution, evaluate, exact_makespan,
                       pack_solutions, two_pass_estimate)  # noqa: F401 (module attribute, as in the reference)

_D, _P = OpKind.DROPOFF, OpKind.PICKUP

DESTROY_OPERATORS = ("random", "worst", "shaw", "cluster", "route", "critical_path")
REPAIR_OPERATORS = ("greedy", "regret2", "regret3", "regretm")
SHAW_TRAVEL_WEIGHT = 9.0
SHAW_TIME_WEIGHT = 3.0
SHAW_AGENT_WEIGHT = 5.0
WORST_POWER = 6.0
_REGRET_K = {"greedy": 0, "regret2": 2, "regret3": 3}
_NEAR_BOTTLENECK = 0.9
_VERIFY_LIMIT = 10


@dataclass
class AlnsParams:
    t0: float = 0.30
    alpha: float = 0.9998
    reheat_factor: float = 0.50
    stagnation_threshold: int = 2000
    weight_interval: int = 100
    reaction: float = 0.1
    sigma1: float = 33.0
    sigma2: float = 9.0
    sigma3: float = 13.0
    min_weight: float = 0.1
    max_iter: int = 20000
    workers_per_pool: int = 32
    pickup_reposition_interval: int = 200
    cross_agent_interval: int = 500
    best_check_interval: int = 1000
    pool_sync_interval: int = 100

    def __post_init__(self):
        if not 0.0 < self.alpha < 1.0:
            raise ValueError("cooling rate must lie in (0, 1)")
        if not self.sigma1 > self.sigma3 > self.sigma2 > 0:
            raise ValueError("scores must satisfy sigma1 > sigma3 > sigma2 > 0")
        for name in ("weight_interval", "pickup_reposition_interval", "cross_agent_interval",
                     "best_check_interval", "pool_sync_interval"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")


@dataclass
class OperatorBank:
    weights: dict
    scores: dict
    attempts: dict

    @classmethod
    def fresh(cls) -> "OperatorBank":
        names = DESTROY_OPERATORS + REPAIR_OPERATORS
        return cls(weights=dict.fromkeys(names, 1.0), scores=dict.fromkeys(names, 0.0),
                   attempts=dict.fromkeys(names, 0))


@dataclass
class AlnsStats:
    iterations: int = 0
    initial_makespan: float = 0.0
    best_trace: list = field(default_factory=list)
    weight_rows: list = field(default_factory=list)
    attempts: dict = field(default_factory=dict)
    accepted: int = 0
    rejected_candidates: int = 0
    reheats: int = 0
    final_temperature: float = 0.0


class EmptySolution(Exception):
    pass


def removal_bounds(n: int) -> tuple:
    """q_max = max(4, n // 20), q_min = max(4, q_max // 2) (alns.py:102-109)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    q_max = max(4, n // 20)
    return max(4, q_max // 2), q_max


def sa_accept(z_candidate: float, z_current: float, temperature: float, rng) -> bool:
    if temperature <= 0:
        raise ValueError("temperature must be positive")
    if z_candidate < z_current:
        return True
    return rng.random() < math.exp(-(z_candidate - z_current) / temperature)


def update_weights(bank: OperatorBank, r: float, min_weight: float = 0.1) -> OperatorBank:
    for name, w in bank.weights.items():
        a = bank.attempts[name]
        avg = bank.scores[name] / a if a else 0.0
        bank.weights[name] = max(min_weight, (1.0 - r) * w + r * avg)
        bank.scores[name] = 0.0
        bank.attempts[name] = 0
    return bank


def roulette_select(names, weights: dict, rng) -> str:
    total = sum(weights[x] for x in names)
    x = rng.random() * total
    acc = 0.0
    for name in names:
        acc += weights[name]
        if x < acc:
            return name
    return names[-1]


def shaw_relatedness(instance, schedule, ci: int, cj: int) -> float:
    r = SHAW_TRAVEL_WEIGHT * instance.d[ci][cj]
    r += SHAW_TIME_WEIGHT * abs(schedule.t_drop[ci] - schedule.t_drop[cj])
    half = SHAW_AGENT_WEIGHT / 2.0
    if schedule.drop_vehicle[ci] != schedule.drop_vehicle[cj]:
        r += half
    if schedule.pickup_vehicle[ci] != schedule.pickup_vehicle[cj]:
        r += half
    return r


# --------------------------------------------------------------------------
# destroy (device: K6)
# --------------------------------------------------------------------------

def destroy(instance, solution: Solution, operator: str, q: int, rng):
    """Remove (at least) q customers with one of the six operators
    (alns.py:182-251), then the capacity cascade of remove_customers
    (insertion.py:379-397); returns (partial Solution, removed list).

    Runs K6 (``vrp_destroy_batch``) on one solution.  ``rng`` must be a
    ``Generator(Philox)`` for draw-for-draw parity: its state goes to the
    device and comes back advanced exactly as the reference's operator
    advances it.  Any other generator is replaced by a Philox stream keyed
    from it (rng.as_philox)."""
    from . import device as Dev
    import torch
    n = instance.n
    if n == 0 or all(not t for t in solution.tours):
        raise EmptySolution("nothing to remove")
    if operator not in DESTROY_OPERATORS:
        raise ValueError(f"unknown destroy operator {operator!r}")
    gen = R.as_philox(rng)
    ops, lens = solution.to_arrays(n)
    state = R.state_to_device(gen)[None]
    r = Dev.destroy_batch(instance, ops[None, :2 * n], lens[None],
                          torch.tensor([Dev.DESTROY_CODES[operator]], dtype=torch.int32),
                          torch.tensor([min(int(q), n)], dtype=torch.int32),
                          min(removal_bounds(n)[0], n), state)
    R.state_from_device(gen, state[0])
    nr = int(r["nremoved"][0].item())
    partial = Solution.from_arrays(r["ops"][0].cpu().numpy(), r["lens"][0].cpu().numpy())
    return partial, [int(c) for c in r["removed"][0, :nr].cpu().numpy()]


# --------------------------------------------------------------------------
# repair (device)
# --------------------------------------------------------------------------

def _repair_scored(instance, partial: Solution, removed, operator: str, rng):
    if operator not in REPAIR_OPERATORS:
        raise ValueError(f"unknown repair operator {operator!r}")
    if not removed:
        return partial, exact_makespan(instance, partial)
    ctx = InsertionContext(instance, partial.tours)
    insertion.reinsert_all(ctx, removed, regret_k=_REGRET_K.get(operator, instance.m), rng=rng)
    sol = ctx.solution()
    try:
        z = exact_makespan(instance, sol)
    except ScheduleError as exc:
        raise RepairFailed(str(exc)) from exc
    return sol, z


def repair(instance, partial: Solution, removed, operator: str, rng) -> Solution:
    if not removed:
        return partial
    return _repair_scored(instance, partial, removed, operator, rng)[0]


# --------------------------------------------------------------------------
# initial solution (host construction + device-scored local search)
# --------------------------------------------------------------------------

def sweep_order(instance) -> list:
    """Customers in the reference's coordinate-free sweep order
    (alns.py:290-298): anchor a = the customer farthest from the depot, b =
    the customer farthest from a (lowest index on ties), then ascending
    (d[a][c] - d[b][c], d[0][c], c)."""
    D = np.asarray(instance.arrays()[0] if hasattr(instance, "arrays") else instance.d, np.float64)
    cs = np.arange(1, instance.n + 1)
    a = 1 + int(np.argmax(D[0, 1:]))  # argmax keeps the first maximum: the lowest customer
    b = 1 + int(np.argmax(D[a, 1:]))
    order = np.lexsort((cs, D[0, cs], D[a, cs] - D[b, cs]))
    return [int(c) for c in cs[order]]


def _balance_sectors(instance, sectors) -> list:
    """Rebalance sector workloads w(c) = 2 d[0][c] + p[c] (alns.py:301-327):
    while some load deviates from the mean by >= 10 %, move the customer of
    the heaviest sector whose move to the lightest lowers the peak load most
    (first such customer in sector order); stop after 2n moves or when no move
    lowers the peak.  Loads are summed with the builtin sum, as there."""
    D = np.asarray(instance.arrays()[0] if hasattr(instance, "arrays") else instance.d, np.float64)
    P = np.asarray(instance.arrays()[1] if hasattr(instance, "arrays") else instance.p, np.float64)
    w = 2.0 * D[0] + P  # w[c] for c = 1..n (w[0] unused)
    secs = [list(x) for x in sectors]
    loads = [sum(float(w[c]) for c in x) for x in secs]
    if not loads:
        return secs
    mean = sum(loads) / len(loads)
    for _ in range(2 * instance.n):
        if mean <= 0 or max(abs(x - mean) for x in loads) < 0.10 * mean:
            break
        arr = np.asarray(loads)
        hi, lo = int(np.argmax(arr)), int(np.argmin(arr))
        if not secs[hi]:
            break
        others = np.delete(arr, [hi, lo])
        rest = others.max() if others.size else -np.inf
        wc = w[np.asarray(secs[hi])]
        peaks = np.maximum(np.maximum(arr[hi] - wc, arr[lo] + wc), rest)
        j = int(np.argmin(peaks))
        if not peaks[j] < arr.max():
            break
        c = secs[hi].pop(j)
        secs[lo].append(c)
        loads[hi] -= float(w[c])
        loads[lo] += float(w[c])
    return secs


def _route_sector(instance, customers) -> list:
    from .brkga import _route_group
    return _route_group(instance, customers)


def _ls_batch(instance, kind, sols):
    from . import localsearch as LS
    n = instance.n
    arrs = [s.to_arrays(n) for s in sols]
    ops = np.stack([o[:2 * n] for o, _ in arrs])
    lens = np.stack([l for _, l in arrs])
    fn = LS.pickup_repositioning_batch if kind == 0 else LS.cross_agent_relocation_batch
    o, l, z = fn(instance, ops, lens)
    o, l = o.cpu().numpy(), l.cpu().numpy()
    return [Solution.from_arrays(o[i], l[i]) for i in range(len(sols))], z


def pickup_repositioning(instance, solution: Solution) -> Solution:
    """Move pickups off (near-)bottleneck vehicles; <= 3 improvement passes
    (alns.py:416-450).  The neighbourhood is built on the device and estimated
    by K2, the best ten verified by K1 (localsearch.py)."""
    return _ls_batch(instance, 0, [solution])[0][0]


def cross_agent_relocation(instance, solution: Solution) -> Solution:
    """Move whole customers off the bottleneck route; <= 3 passes
    (alns.py:453-487), device-built neighbourhood (localsearch.py)."""
    if instance.m == 1:
        return solution
    return _ls_batch(instance, 1, [solution])[0][0]


def construct_initial(instance, seed: int = 0) -> Solution:
    """Sweep sectors, balance, greedy-route each, then the local-search pair
    until no improvement (alns.py:369-390)."""
    m, n = instance.m, instance.n
    order = sweep_order(instance)
    sizes = [n // m + (1 if i < n % m else 0) for i in range(m)]
    sectors, at = [], 0
    for s in sizes:
        sectors.append(order[at:at + s])
        at += s
    sectors = _balance_sectors(instance, sectors)
    sol = Solution.from_lists([_route_sector(instance, sec) for sec in sectors])
    evaluate(instance, sol)
    for _ in range(10):
        z = evaluate(instance, sol).makespan
        sol = pickup_repositioning(instance, sol)
        sol = cross_agent_relocation(instance, sol)
        if evaluate(instance, sol).makespan >= z - 1e-9:
            break
    return sol


# --------------------------------------------------------------------------
# main loop
# --------------------------------------------------------------------------

def _rng_for(seed: int):
    return R.philox_generator(seed, R.ALNS_STREAM)


def worker_seed(seed: int, worker: int) -> int:
    return int(np.random.SeedSequence([seed, worker]).generate_state(1)[0])


class _PoolShare:
    """A pool's shared incumbent (alns.py:503-533 semantics).  Workers of a
    pool advance in lockstep on one host thread, so no lock is needed.
    ``offer`` keeps strictly better solutions (remembering the source
    worker), ``poll`` returns the incumbent to every other worker, and
    ``merge`` moves a strictly better incumbent across two shares (the
    receiver forgets the source)."""

    def __init__(self):
        self.best_z, self.best_sol, self.src = math.inf, None, None

    def offer(self, worker: int, z: float, sol: Solution) -> None:
        if z < self.best_z:
            self.best_z, self.best_sol, self.src = z, sol, worker

    def poll(self, worker: int):
        if self.best_sol is None or self.src == worker:
            return None
        return self.best_z, self.best_sol

    def merge(self, other: "_PoolShare") -> None:
        if self.best_z < other.best_z:
            other.best_z, other.best_sol, other.src = self.best_z, self.best_sol, None
        elif other.best_z < self.best_z:
            self.best_z, self.best_sol, self.src = other.best_z, other.best_sol, None


class _Worker:
    """One ALNS trajectory (alns.py:536-640) split into phases so that many
    workers can share the device launches of an iteration (host engine), or
    so that the device engine can hand the host its boundary steps."""

    def __init__(self, instance, params: AlnsParams, seed: int, initial=None, share=None,
                 global_share=None, worker_id: int = 0, rng=None):
        self.instance, self.params = instance, params
        self.rng = rng if rng is not None else _rng_for(seed)
        self._cur_arr = self._best_arr = None
        self.current = initial if initial is not None else construct_initial(instance, seed)
        self.z = exact_makespan(instance, self.current)
        self.best, self.z_best = self.current, self.z
        self.temperature = params.t0 * self.z
        self.t_init = self.temperature
        self.bank = OperatorBank.fresh()
        self.stagnation = 0
        self.best_it = 0
        q_min, q_max = removal_bounds(instance.n)
        q_min, q_max = min(q_min, instance.n), min(q_max, instance.n)
        self.stats = AlnsStats(initial_makespan=self.z)
        self.stats.best_trace.append((0, self.z_best))
        self.q_draws = (self.rng.integers(q_min, q_max + 1, size=params.max_iter)
                        if params.max_iter else [])
        self.share, self.global_share, self.worker_id = share, global_share, worker_id

    # current / best are materialised lazily from device arrays (device engine)
    @property
    def current(self):
        if self._current is None:
            self._current = Solution.from_arrays(*self._cur_arr)
        return self._current

    @current.setter
    def current(self, sol):
        self._current, self._cur_arr, self.cur_dirty = sol, None, True

    @property
    def best(self):
        if self._best is None:
            self._best = Solution.from_arrays(*self._best_arr)
        return self._best

    @best.setter
    def best(self, sol):
        self._best, self._best_arr, self.best_dirty = sol, None, True

    def _found_best(self, sol, value, it):
        self.best, self.z_best = sol, value
        self.best_it = it
        self.stagnation = 0
        self.stats.best_trace.append((it, value))
        if self.share is not None:
            self.share.offer(self.worker_id, value, sol)

    # phase 1: operator selection + destroy (host engine)
    def propose(self, it: int):
        bank, rng = self.bank, self.rng
        self.dname = roulette_select(DESTROY_OPERATORS, bank.weights, rng)
        self.rname = roulette_select(REPAIR_OPERATORS, bank.weights, rng)
        bank.attempts[self.dname] += 1
        bank.attempts[self.rname] += 1
        q = int(self.q_draws[it - 1])
        try:
            self.partial, self.removed = destroy(self.instance, self.current, self.dname, q, rng)
            self.failed = False
        except (RepairFailed, ScheduleError):
            self.failed = True
        if self.rname not in REPAIR_OPERATORS:
            raise ValueError(f"unknown repair operator {self.rname!r}")
        return not self.failed

    # phase 3: acceptance + bookkeeping, given the repaired candidate
    def conclude(self, it: int, cand, z_cand, failed: bool):
        self.accept(it, cand, z_cand, failed)
        self.post(it)

    def accept(self, it: int, cand, z_cand, failed: bool):
        """alns.py:577-611 -- what the device engine runs inside the kernel."""
        p, bank = self.params, self.bank
        if failed:
            self.stats.rejected_candidates += 1
        elif z_cand < self.z:
            self.current, self.z = cand, z_cand
            bank.scores[self.dname] += p.sigma2
            bank.scores[self.rname] += p.sigma2
            self.stats.accepted += 1
            if z_cand < self.z_best:
                bank.scores[self.dname] += p.sigma1 - p.sigma2
                bank.scores[self.rname] += p.sigma1 - p.sigma2
                self._found_best(cand, z_cand, it)
        elif self.temperature > 0 and self.rng.random() < math.exp(-(z_cand - self.z) / self.temperature):
            self.current, self.z = cand, z_cand
            bank.scores[self.dname] += p.sigma3
            bank.scores[self.rname] += p.sigma3
            self.stats.accepted += 1
        self.temperature *= p.alpha
        self.stagnation += 1
        if self.stagnation >= p.stagnation_threshold and self.temperature < 0.01 * self.t_init:
            self.temperature = p.reheat_factor * p.t0 * self.z_best
            self.stagnation = 0
            self.stats.reheats += 1
        if it % p.weight_interval == 0:
            update_weights(bank, p.reaction, p.min_weight)
            self._weight_row(it, self.z_best, self.temperature, [bank.weights[k] for k in bank.weights])

    def _weight_row(self, it, z_best, temperature, weights):
        self.stats.weight_rows.append({"iteration": it, "best_makespan": z_best,
                                       "temperature": temperature,
                                       **{f"w_{k}": w for k, w in zip(self.bank.weights, weights)}})

    def post(self, it: int):
        """alns.py:612-640: local search, pool share polling and merging."""
        p, inst = self.params, self.instance
        cache = getattr(self, "ls_cache", None) or {}
        self.ls_cache = None
        if it % p.pickup_reposition_interval == 0:
            if "pickup" in cache:
                improved, z_new = cache["pickup"]
            else:
                improved = pickup_repositioning(inst, self.current)
                z_new = exact_makespan(inst, improved)
            if z_new < self.z:
                self.current, self.z = improved, z_new
                if z_new < self.z_best:
                    self._found_best(improved, z_new, it)
        if it % p.cross_agent_interval == 0:
            if "cross" in cache:
                improved, z_new = cache["cross"]
            else:
                improved = cross_agent_relocation(inst, self.current)
                z_new = exact_makespan(inst, improved)
            if z_new < self.z:
                self.current, self.z = improved, z_new
                if z_new < self.z_best:
                    self._found_best(improved, z_new, it)
        if self.share is not None and it % p.best_check_interval == 0:
            got = self.share.poll(self.worker_id)
            if got is not None and got[0] < self.z:
                self.z, self.current = got[0], got[1]
                if self.z < self.z_best:
                    self.best, self.z_best = self.current, self.z
                    self.stats.best_trace.append((it, self.z))
        if self.share is not None and self.global_share is not None and it % p.pool_sync_interval == 0:
            self.share.merge(self.global_share)

    def host_step(self, it: int) -> bool:
        """Does post(it) have anything to do?"""
        p = self.params
        return (it % p.pickup_reposition_interval == 0 or it % p.cross_agent_interval == 0
                or (self.share is not None and (it % p.best_check_interval == 0 or (
                    self.global_share is not None and it % p.pool_sync_interval == 0))))

    # device engine: worker <-> vrp_alns_worker record
    def to_record(self, rec):
        rec["rng"] = R.state_bytes(self.rng)
        rec["z"], rec["z_best"] = self.z, self.z_best
        rec["temperature"], rec["t_init"] = self.temperature, self.t_init
        names = list(self.bank.weights)
        rec["weights"] = [self.bank.weights[k] for k in names]
        rec["scores"] = [self.bank.scores[k] for k in names]
        rec["attempts"] = [self.bank.attempts[k] for k in names]
        rec["stagnation"] = self.stagnation
        rec["accepted"] = self.stats.accepted
        rec["rejected"] = self.stats.rejected_candidates
        rec["reheats"] = self.stats.reheats
        rec["best_it"] = self.best_it
        rec["n_trace"] = rec["n_rows"] = 0

    def from_record(self, rec, trace, rows, cur_arr, best_arr):
        R.set_state_bytes(self.rng, rec["rng"])
        self.z, self.z_best = float(rec["z"]), float(rec["z_best"])
        self.temperature, self.t_init = float(rec["temperature"]), float(rec["t_init"])
        names = list(self.bank.weights)
        for j, k in enumerate(names):
            self.bank.weights[k] = float(rec["weights"][j])
            self.bank.scores[k] = float(rec["scores"][j])
            self.bank.attempts[k] = int(rec["attempts"][j])
        self.stagnation = int(rec["stagnation"])
        self.stats.accepted = int(rec["accepted"])
        self.stats.rejected_candidates = int(rec["rejected"])
        self.stats.reheats = int(rec["reheats"])
        self.best_it = int(rec["best_it"])
        self.stats.best_trace.extend(trace)
        for it, vals in rows:
            self._weight_row(it, vals[0], vals[1], vals[2:])
        self._current, self._cur_arr, self.cur_dirty = None, cur_arr, False
        if trace:
            self._best, self._best_arr, self.best_dirty = None, best_arr, False

    def finish(self):
        self.stats.iterations = self.params.max_iter
        self.stats.attempts = dict(self.bank.attempts)
        self.stats.final_temperature = self.temperature
        return self.best, self.stats


class _DeviceWorkers:
    """Device-resident state of a list of workers driven by vrp_alns_iterate
    (csrc/alns_step.cu).  The kernel runs stretches of iterations; the host
    steps in only at iterations where post() has work (local search, share
    polling/merging), in worker order, exactly where the sequential loop
    would."""

    def __init__(self, instance, params: AlnsParams, workers):
        import torch
        from . import device as DV
        self.DV, self.torch = DV, torch
        self.instance, self.params, self.workers = instance, params, workers
        n, m, W = instance.n, instance.m, len(workers)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.cparams = DV.AlnsParamsC(
            t0=params.t0, alpha=params.alpha, reheat_factor=params.reheat_factor,
            reaction=params.reaction, sigma1=params.sigma1, sigma2=params.sigma2,
            sigma3=params.sigma3, min_weight=params.min_weight,
            stagnation_threshold=params.stagnation_threshold, weight_interval=params.weight_interval,
            q_min=min(removal_bounds(n)[0], n), reserved=0)
        self.rec = np.zeros(W, DV.ALNS_WORKER_DTYPE)
        cur = [w.current.to_arrays(n) for w in workers]
        best = [w.best.to_arrays(n) for w in workers]
        self.g_cur_ops = torch.from_numpy(np.stack([o[:2 * n] for o, _ in cur])).to(self.dev)
        self.g_cur_lens = torch.from_numpy(np.stack([l for _, l in cur])).to(self.dev)
        self.g_best_ops = torch.from_numpy(np.stack([o[:2 * n] for o, _ in best])).to(self.dev)
        self.g_best_lens = torch.from_numpy(np.stack([l for _, l in best])).to(self.dev)
        self.g_q = torch.from_numpy(np.stack([np.asarray(w.q_draws, np.int32) for w in workers])).to(self.dev)
        self.g_rec = torch.empty((W, DV.ALNS_WORKER_DTYPE.itemsize), dtype=torch.uint8, device=self.dev)
        self._cap = 0
        for w in workers:
            w.cur_dirty = w.best_dirty = False
        self.push()

    def _buffers(self, length):
        if length > self._cap:
            torch, W = self.torch, len(self.workers)
            self._cap = length
            rcap = length // self.params.weight_interval + 2
            self.t_it = torch.empty((W, length), dtype=torch.int32, device=self.dev)
            self.t_z = torch.empty((W, length), dtype=torch.float64, device=self.dev)
            self.r_it = torch.empty((W, rcap), dtype=torch.int32, device=self.dev)
            self.r_val = torch.empty((W, rcap, 12), dtype=torch.float64, device=self.dev)

    def push(self):
        n = self.instance.n
        for i, w in enumerate(self.workers):
            w.to_record(self.rec[i])
            if w.cur_dirty:
                o, l = w.current.to_arrays(n)
                self.g_cur_ops[i].copy_(self.torch.from_numpy(o[:2 * n]))
                self.g_cur_lens[i].copy_(self.torch.from_numpy(l))
                w.cur_dirty = False
            if w.best_dirty:
                o, l = w.best.to_arrays(n)
                self.g_best_ops[i].copy_(self.torch.from_numpy(o[:2 * n]))
                self.g_best_lens[i].copy_(self.torch.from_numpy(l))
                w.best_dirty = False
        self.g_rec.copy_(self.torch.from_numpy(self.rec.view(np.uint8).reshape(len(self.workers), -1)))

    def run(self, a: int, b: int):
        """Iterations a..b on the device, then pull the state back."""
        self._buffers(b - a + 1)
        self.DV.alns_iterate(self.instance, self.cparams, self.g_rec, self.g_cur_ops, self.g_cur_lens,
                             self.g_best_ops, self.g_best_lens, self.g_q, a, b, self.t_it, self.t_z,
                             self.r_it, self.r_val)
        rec = self.g_rec.cpu().numpy().view(self.DV.ALNS_WORKER_DTYPE).reshape(-1)
        t_it, t_z = self.t_it.cpu().numpy(), self.t_z.cpu().numpy()
        r_it, r_val = self.r_it.cpu().numpy(), self.r_val.cpu().numpy()
        cur_o, cur_l = self.g_cur_ops.cpu().numpy(), self.g_cur_lens.cpu().numpy()
        best_o, best_l = self.g_best_ops.cpu().numpy(), self.g_best_lens.cpu().numpy()
        improved = []
        for i, w in enumerate(self.workers):
            nt, nr = int(rec[i]["n_trace"]), int(rec[i]["n_rows"])
            trace = [(int(t_it[i, j]), float(t_z[i, j])) for j in range(nt)]
            rows = [(int(r_it[i, j]), [float(x) for x in r_val[i, j]]) for j in range(nr)]
            w.from_record(rec[i], trace, rows, (cur_o[i], cur_l[i]), (best_o[i], best_l[i]))
            if nt:
                improved.append(i)
        self.rec = rec.copy()
        return improved

    def local_search(self, b: int):
        """The local-search pair of post(b) for every worker in two batched
        passes (localsearch.py); results are handed to post() in ls_cache.
        The cross pass starts from the pickup pass's result exactly when
        post() will have adopted it (strict improvement)."""
        from . import localsearch as LS
        p, ws, inst = self.params, self.workers, self.instance
        do_p = b % p.pickup_reposition_interval == 0
        do_c = b % p.cross_agent_interval == 0
        if not (do_p or do_c):
            return
        n = inst.n
        ops, lens = self.g_cur_ops, self.g_cur_lens
        for w in ws:
            w.ls_cache = {}
        if do_p:
            o, l, z = LS.pickup_repositioning_batch(inst, ops, lens)
            on, ln = o.cpu().numpy(), l.cpu().numpy()
            for i, w in enumerate(ws):
                w.ls_cache["pickup"] = (Solution.from_arrays(on[i], ln[i]), float(z[i]))
            adopt = self.torch.from_numpy(np.array([float(z[i]) < w.z for i, w in enumerate(ws)])).to(o.device)
            ops = self.torch.where(adopt[:, None], o, ops)
            lens = self.torch.where(adopt[:, None], l, lens)
        if do_c and inst.m > 1:
            o, l, z = LS.cross_agent_relocation_batch(inst, ops, lens)
            on, ln = o.cpu().numpy(), l.cpu().numpy()
            for i, w in enumerate(ws):
                w.ls_cache["cross"] = (Solution.from_arrays(on[i], ln[i]), float(z[i]))

    def drive(self, stop=None, max_stretch: int | None = None, on_boundary=None):
        """Run to max_iter (or until ``stop()`` is true at a stretch end);
        ``on_boundary(b)`` runs after every worker's post(b)."""
        p, workers = self.params, self.workers
        pooled = workers[0].share is not None
        it = 1
        while it <= p.max_iter:
            b = it
            while (b < p.max_iter and not workers[0].host_step(b)
                   and (max_stretch is None or b - it + 1 < max_stretch)):
                b += 1
            if pooled:
                # offers made before b reach the shares before anyone polls at b,
                # in (iteration, worker) order; b's own offers interleave with post(b)
                if b > it:
                    pre = self.run(it, b - 1)
                    for i in sorted(pre, key=lambda i: (workers[i].best_it, i)):
                        w = workers[i]
                        w.share.offer(w.worker_id, w.z_best, w.best)
                at_b = set(self.run(b, b))
                self.local_search(b)
                for i, w in enumerate(workers):
                    if i in at_b:
                        w.share.offer(w.worker_id, w.z_best, w.best)
                    w.post(b)
            else:
                self.run(it, b)
                self.local_search(b)
                for w in workers:
                    w.post(b)
            if on_boundary is not None:
                on_boundary(b)
            self.push()
            self.iterations = b
            it = b + 1
            if stop is not None and stop():
                break


def _repair_many(instance, workers):
    """Repair every live worker's partial in one K5 launch, score in one K1
    launch; returns [(cand, z, failed)] aligned with ``workers``."""
    from .device import makespan_batch
    live = [w for w in workers if not w.failed]
    out = {id(w): (None, 0.0, True) for w in workers}
    need = [w for w in live if w.removed]
    for w in live:
        if not w.removed:  # nothing removed: the partial is the candidate
            try:
                out[id(w)] = (w.partial, exact_makespan(instance, w.partial), False)
            except ScheduleError:
                out[id(w)] = (None, 0.0, True)
    if need:
        parts, lens = pack_solutions(instance, [w.partial for w in need])
        o, l, st = insertion.reinsert_batch(
            instance, parts, lens, [w.removed for w in need],
            [_REGRET_K.get(w.rname, instance.m) for w in need], [w.rng for w in need])
        ok = np.flatnonzero(st == 0)
        if ok.size:
            r = makespan_batch(instance, o[ok], l[ok], mode=0)
            z = r["z"].cpu().numpy()
            zs = r["status"].cpu().numpy()
        for j, w in enumerate(need):
            if st[j] != 0:
                continue
            k = int(np.searchsorted(ok, j))
            if zs[k] != 0:
                continue
            out[id(w)] = (Solution.from_arrays(o[j], l[j]), float(z[k]), False)
    return [out[id(w)] for w in workers]


def run_alns(instance, params: AlnsParams, seed: int, initial: Solution | None = None,
             share: _PoolShare | None = None, global_share: _PoolShare | None = None,
             worker_id: int = 0, rng=None, engine: str = "device"):
    """Single trajectory (alns.py:536-640); returns (best Solution, AlnsStats).
    engine "device": the whole loop body runs in vrp_alns_iterate; "host":
    destroy/acceptance on the host, repair + scoring batched on the device."""
    w = _Worker(instance, params, seed, initial, share, global_share, worker_id, rng=rng)
    _drive([w], engine)
    return w.finish()


def _drive(workers, engine: str, on_boundary=None):
    if engine == "device":
        if workers[0].params.max_iter:
            _DeviceWorkers(workers[0].instance, workers[0].params, workers).drive(on_boundary=on_boundary)
        return
    if engine != "host":
        raise ValueError(f"unknown engine {engine!r}")
    instance, params = workers[0].instance, workers[0].params
    for it in range(1, params.max_iter + 1):
        for w in workers:
            w.propose(it)
        results = _repair_many(instance, workers)
        for w, (cand, z, failed) in zip(workers, results):
            w.conclude(it, cand, z, failed)
        if on_boundary is not None and workers[0].host_step(it):
            on_boundary(it)


def run_pool(instance, params: AlnsParams, pool_size: int, seed: int,
             initial: Solution | None = None, engine: str = "device"):
    """pool_size workers with derived seeds (alns.py:643-685).  Workers offer
    and poll their pool's incumbent in worker order (deterministic; the
    reference's threads interleave nondeterministically).  engine "device":
    one warp per worker inside vrp_alns_iterate; "host": lockstep iterations
    with one batched repair + one batched scoring launch each."""
    if pool_size < 1:
        raise ValueError("pool_size must be >= 1")
    if pool_size == 1:
        best, stats = run_alns(instance, params, worker_seed(seed, 0), initial=initial, engine=engine)
        return best, {"workers": 1, "pools": 1, "best_makespan": evaluate(instance, best).makespan,
                      "worker_stats": [stats]}
    if initial is None:
        initial = construct_initial(instance)
    n_pools = (pool_size + params.workers_per_pool - 1) // params.workers_per_pool
    pools = [_PoolShare() for _ in range(n_pools)]
    global_share = _PoolShare() if n_pools > 1 else None
    workers = [_Worker(instance, params, worker_seed(seed, i), initial,
                       pools[i // params.workers_per_pool], global_share, i)
               for i in range(pool_size)]
    _drive(workers, engine)
    results = [w.finish() for w in workers]
    best, z_best = None, math.inf
    for sol, _ in results:
        z = evaluate(instance, sol).makespan
        if z < z_best:
            best, z_best = sol, z
    for pool in pools:
        if pool.best_sol is not None and pool.best_z < z_best:
            best, z_best = pool.best_sol, pool.best_z
    return best, {"workers": pool_size, "pools": n_pools, "best_makespan": z_best,
                  "worker_stats": [st for _, st in results]}


# --------------------------------------------------------------------------
# multi-GPU pools: pools sharded over ranks, the global share
# kept consistent by a min-all-reduce + broadcast at every pool_sync boundary
# --------------------------------------------------------------------------

def _dist_world(group):
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def sync_pool_share(instance, share: _PoolShare, group=None) -> None:
    """Make ``share`` the best over all ranks: min-all-reduce of its makespan,
    the lowest rank among equals wins, its routes are broadcast (2n + m int32).
    The result is the same on every rank (src = None, as after merge())."""
    import torch
    import torch.distributed as dist
    rank, world = _dist_world(group)
    if world < 2:
        return
    dev = (torch.device("cuda", torch.cuda.current_device())
           if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    z = torch.tensor([share.best_z], dtype=torch.float64, device=dev)
    dist.all_reduce(z, op=dist.ReduceOp.MIN, group=group)
    zmin = float(z.item())
    if zmin == math.inf:
        return
    cand = torch.tensor([rank if share.best_z == zmin else world], dtype=torch.int64, device=dev)
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    winner = int(cand.item())
    n, m = instance.n, instance.m
    buf = torch.zeros(2 * n + m, dtype=torch.int32, device=dev)
    if rank == winner:
        o, l = share.best_sol.to_arrays(n)
        buf[:2 * n] = torch.from_numpy(o[:2 * n])
        buf[2 * n:] = torch.from_numpy(l)
    src = dist.get_global_rank(group, winner) if group is not None else winner
    dist.broadcast(buf, src=src, group=group)
    arr = buf.cpu().numpy()
    share.best_z, share.src = zmin, None
    share.best_sol = Solution.from_arrays(arr[:2 * n], arr[2 * n:])


def run_pool_distributed(instance, params: AlnsParams, pool_size: int, seed: int,
                         initial: Solution | None = None, group=None, engine: str = "device"):
    """run_pool with its pools sharded over the ranks of ``group`` (pool p on
    rank p % world).  Workers keep their global ids and seeds; every rank's
    copy of the global share is re-synchronised (sync_pool_share) after each
    pool_sync_interval boundary, so a pool merges with the best of all GPUs
    as of the previous boundary.  Every rank returns the same result."""
    rank, world = _dist_world(group)
    wpp = params.workers_per_pool
    n_pools = (pool_size + wpp - 1) // wpp
    if world > n_pools:
        raise ValueError(f"{world} ranks need at least {world} pools (pool_size / workers_per_pool)")
    if initial is None:
        initial = construct_initial(instance)
    pools = {p: _PoolShare() for p in range(n_pools) if p % world == rank}
    global_share = _PoolShare() if (n_pools > 1 or world > 1) else None
    workers = [_Worker(instance, params, worker_seed(seed, i), initial, pools[i // wpp], global_share, i)
               for i in range(pool_size) if (i // wpp) % world == rank]

    def boundary(b):
        if global_share is not None and b % params.pool_sync_interval == 0:
            sync_pool_share(instance, global_share, group)

    _drive(workers, engine, on_boundary=boundary)
    results = [w.finish() for w in workers]
    final = _PoolShare()
    for sol, _ in results:
        final.offer(-1, evaluate(instance, sol).makespan, sol)
    for pool in pools.values():
        if pool.best_sol is not None:
            final.offer(-1, pool.best_z, pool.best_sol)
    sync_pool_share(instance, final, group)
    return final.best_sol, {"workers": pool_size, "pools": n_pools, "ranks": world,
                            "local_workers": len(workers), "best_makespan": final.best_z,
                            "worker_stats": [st for _, st in results]}
