"""Experiment harness -- the reference's experiment grid and result CSV
(``vrp_rpd.bench``: ``ExperimentConfig``, ``ResultRow``, ``write_rows_csv`` /
``read_rows_csv``, ``run_experiment``; bench.py:130-258) for the GPU
methods, with throughput columns.

The grid is (instance x variant kind x replicate x method).  Rows keep the
reference's nine fields first, in its order and float encoding (``repr``, so
the CSV round-trips losslessly), then add:
  budget_s         wall-clock budget of the "budget" method (0 otherwise)
  k1_evals_per_s   exact-makespan evaluations/s of K1 on that instance
                   (65,536 decoded candidates, measured once per instance)
  device           the GPU the row ran on
The reference's paired statistics and report rendering (Wilcoxon, Cohen's
d, comparison tables) are presentation, not the hot path, and stay out of
scope.

Methods: "alns" (run_pool / run_alns), "pipeline" (the reference's
ALNS -> warm-started BRKGA, reusing the cell's ALNS incumbent like the
reference), "polish" (construct_initial + device two_opt_improve to a local
optimum), "budget" (pipeline.run_pipeline_budget for ``budget_s``)."""
from __future__ import annotations

import csv
import time
from dataclasses import dataclass, field
from pathlib import Path

from . import alns as A
from . import brkga as B
from .instance import VariantSpec, build_instance, load_tsplib_file
from .schedule import coordination_metrics, evaluate

METHODS = ("alns", "pipeline", "polish", "budget")
DEFAULT_REPLICATES = {"base": 1, "2x": 1, "5x": 1, "1R10": 10, "1R20": 10}


@dataclass
class ExperimentConfig:
    instance_files: list
    kinds: tuple = ("base", "2x", "5x", "1R10", "1R20")
    replicates: dict = field(default_factory=lambda: dict(DEFAULT_REPLICATES))
    methods: tuple = METHODS
    seed: int = 42
    alns_params: A.AlnsParams = field(default_factory=A.AlnsParams)
    brkga_params: B.BrkgaParams = field(default_factory=B.BrkgaParams)
    pool_size: int = 1
    budget_s: float = 60.0
    out_dir: str | None = None


@dataclass
class ResultRow:
    instance: str
    variant: str
    replicate: int
    method: str
    makespan: float
    runtime: float
    cross_agent_pct: float
    interleaved_pct: float
    seed: int
    budget_s: float = 0.0
    k1_evals_per_s: float = 0.0
    device: str = ""

    FIELDS = ("instance", "variant", "replicate", "method", "makespan",
              "runtime", "cross_agent_pct", "interleaved_pct", "seed")
    EXTRA = ("budget_s", "k1_evals_per_s", "device")

    def as_list(self):
        return [getattr(self, f) for f in self.FIELDS + self.EXTRA]


def write_rows_csv(rows, path) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(ResultRow.FIELDS + ResultRow.EXTRA)
        for row in sorted(rows, key=lambda r: (r.instance, r.variant, r.replicate, r.method)):
            w.writerow([repr(x) if isinstance(x, float) else x for x in row.as_list()])


def read_rows_csv(path) -> list:
    rows = []
    with open(path, newline="", encoding="utf-8") as fh:
        for rec in csv.DictReader(fh):
            rows.append(ResultRow(
                instance=rec["instance"], variant=rec["variant"], replicate=int(rec["replicate"]),
                method=rec["method"], makespan=float(rec["makespan"]), runtime=float(rec["runtime"]),
                cross_agent_pct=float(rec["cross_agent_pct"]),
                interleaved_pct=float(rec["interleaved_pct"]), seed=int(rec["seed"]),
                budget_s=float(rec.get("budget_s") or 0.0),
                k1_evals_per_s=float(rec.get("k1_evals_per_s") or 0.0),
                device=rec.get("device", "")))
    return rows


def k1_rate(instance, count: int = 1 << 16, seed: int = 0) -> float:
    """Exact-makespan evaluations/s of K1 over ``count`` decoded candidates."""
    import torch
    from . import device as DV
    g = torch.rand((count, 4 * instance.n), dtype=torch.float64, device="cuda",
                   generator=torch.Generator("cuda").manual_seed(seed))
    dec = DV.decode_batch(instance, g, op_dtype=torch.int16)
    out = {}
    DV.makespan_batch(instance, dec["ops"], dec["lens"], out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        DV.makespan_batch(instance, dec["ops"], dec["lens"], out=out)
    e1.record()
    torch.cuda.synchronize()
    return 3 * count / (e0.elapsed_time(e1) / 1e3)


def _run_method(instance, method: str, config: ExperimentConfig, cache: dict):
    from . import baselines as BL
    from .pipeline import run_pipeline, run_pipeline_budget
    if method == "alns":
        if "alns" not in cache:
            if config.pool_size > 1:
                cache["alns"], _ = A.run_pool(instance, config.alns_params, config.pool_size, config.seed)
            else:
                cache["alns"], _ = A.run_alns(instance, config.alns_params, config.seed)
        return cache["alns"]
    if method == "pipeline":
        inc = cache.get("alns") or _run_method(instance, "alns", config, cache)
        sol, _ = run_pipeline(instance, config.alns_params, config.brkga_params, config.seed,
                              config.pool_size, incumbent=inc)
        return sol
    if method == "polish":
        return BL.two_opt_improve(instance, A.construct_initial(instance, config.seed), move_budget=10**15)
    if method == "budget":
        sol, _, _ = run_pipeline_budget(instance, config.budget_s, seed=config.seed)
        return sol
    raise ValueError(f"unknown method {method!r}")


def run_experiment(config: ExperimentConfig):
    """Run the grid; per-cell failures are recorded and skipped (bench.py:232-258).
    Returns (rows, failures)."""
    import torch
    dev_name = torch.cuda.get_device_name(torch.cuda.current_device())
    rows, failures = [], []
    for path in config.instance_files:
        raw = load_tsplib_file(path)
        for kind in config.kinds:
            for rep in range(config.replicates.get(kind, 1)):
                inst = build_instance(raw, VariantSpec(kind, config.seed, rep))
                rate = k1_rate(inst)
                cache: dict = {}
                for method in config.methods:
                    t0 = time.perf_counter()
                    try:
                        sol = _run_method(inst, method, config, cache)
                        sched = evaluate(inst, sol)
                        met = coordination_metrics(inst, sol, sched)
                    except Exception as exc:  # cell failure; the run continues
                        failures.append((raw.name, kind, rep, method, str(exc)))
                        continue
                    rows.append(ResultRow(raw.name, kind, rep, method, sched.makespan,
                                          time.perf_counter() - t0, met.cross_agent_pct,
                                          met.interleaved_pct, config.seed,
                                          config.budget_s if method == "budget" else 0.0, rate, dev_name))
    if config.out_dir:
        out = Path(config.out_dir)
        out.mkdir(parents=True, exist_ok=True)
        write_rows_csv(rows, out / "results.csv")
    return rows, failures
