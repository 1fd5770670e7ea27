"""Headline benchmark: candidate makespan evaluations/s at n = 999 (dsj1000-derived, 1R20).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step = one launch of K1 (exact_makespan, csrc/makespan.cu) over this rank's
whole batch of N_CAND candidates, which are decoded (K3, untimed setup) from
seeded uniform random chromosomes, so every candidate is feasible and unique.
The batch (2^20 x 1998 int16 ops = 4.2 GB) is far larger than the 126 MB L2, so
no flush is needed between steps.  Multi-GPU: one process per GPU (torchrun),
each rank scores its own candidates (weak scaling, no data-path collective);
time = max over ranks of the CUDA-event time.

``--impl reference`` times the reference algorithm on the host CPU: the C
restatement in oracle/ (the reference itself is pure Python and not built),
with every host thread, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests" / "golden"))

CONFIG = "dsj1000"
METRIC = "candidate makespan evals/sec at n=1000"
UNIT = "evals/s"


def algorithmic_bytes_per_eval(n: int, m: int) -> int:
    """ops 4*2n + lens 4m + d gathers 8*(2n+m) + p gathers 8n + 12 B out."""
    return 4 * 2 * n + 4 * m + 8 * (2 * n + m) + 8 * n + 12


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        doc = json.loads(p.read_text())
        return float(doc["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting", 0x10: "sync_boost", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference_rate(inst, ops, lens, threads: int, min_seconds: float):
    """Oracle (C restatement of schedule.exact_makespan) on host threads."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    done = 0
    while True:
        O.makespan_batch(inst, ops, lens, mode="exact", threads=threads)
        done += ops.shape[0]
        el = time.perf_counter() - t0
        if el >= min_seconds:
            return done / el, done, el


def make_candidates(inst, count: int, seed: int, device, chunk: int = 1 << 16):
    """Decode `count` seeded random chromosomes on the GPU (K3) -> int16 ops."""
    import torch
    from paper_2602_23685_b200 import device as D
    n, m = inst.n, inst.m
    ops = torch.empty((count, 2 * n), dtype=torch.int16, device=device)
    lens = torch.empty((count, m), dtype=torch.int32, device=device)
    z = torch.empty(count, dtype=torch.float64, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        genes = torch.rand((e - s, 4 * n), dtype=torch.float64, device=device, generator=gen)
        out = {"ops": ops[s:e], "lens": lens[s:e]}
        r = D.decode_batch(inst, genes, out=out)
        z[s:e] = r["makespan"]
        del genes
    return ops, lens, z


def extra_rates(device, ops, lens, decode_ms, n_dec, pipeline_seconds=30.0):
    """Secondary §8 throughputs on this GPU (not the headline): K3 decodes/s
    (the bench set-up, CUDA-event timed), BRKGA generations/s at paper scale
    (N_p = 30,000) on the a280 island config and dsj1000, ALNS repairs/s
    (K5, 1024 instances) and device-resident ALNS iterations/s on the eil51
    ALNS config."""
    import torch
    from oracle import oracle as O
    import inputs as I
    from paper_2602_23685_b200 import brkga as B
    from paper_2602_23685_b200 import insertion as INS
    from paper_2602_23685_b200.configs import config_instance
    # K3 decodes/s on a warm GPU: 65,536 uniform random dsj1000 chromosomes
    dsj = config_instance("dsj1000")
    from paper_2602_23685_b200 import device as D
    g = torch.rand((65536, 4 * dsj.n), dtype=torch.float64, device=device,
                   generator=torch.Generator(device=device).manual_seed(77))
    D.decode_batch(dsj, g[:4096], want_solution=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    D.decode_batch(dsj, g, want_solution=False)
    e1.record()
    torch.cuda.synchronize()
    out = {"decodes_per_s_dsj1000_random": 65536 / (e0.elapsed_time(e1) / 1e3),
           "bench_setup_decodes_per_s": n_dec / (decode_ms / 1e3)}
    del g
    for key in ("a280", "dsj1000"):
        # generations/s of the device loop: (10 - 2) generations over the
        # difference of two runs, so the population set-up cancels out
        inst = config_instance(key)
        B.run_brkga(inst, B.BrkgaParams(population=30000, generations=1), seed=0)  # warm
        el = {}
        for T in (2, 10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            B.run_brkga(inst, B.BrkgaParams(population=30000, generations=T), seed=1)
            torch.cuda.synchronize()
            el[T] = time.perf_counter() - t0
        out[f"brkga_generations_per_s_{key}_Np30000"] = 8 / (el[10] - el[2])
        out[f"brkga_setup_plus_2_generations_s_{key}"] = el[2]
    inst = config_instance("eil51")
    cnt = 1024
    genes = I.chromosomes(inst.n, cnt, (7, 7))
    dec = O.decode_batch(inst, genes)
    parts, plens, rem = [], [], []
    for i in range(cnt):
        pick = I.philox(8, i).choice(np.arange(1, inst.n + 1), size=5, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
    parts, plens = np.stack(parts), np.stack(plens)
    rks = [(0, 2, 3, inst.m)[i % 4] for i in range(cnt)]
    # warm-up with the full batch (the first call of a size pays the scratch pool growth)
    INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(9, i) for i in range(cnt)])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(9, i) for i in range(cnt)])
    torch.cuda.synchronize()
    out["alns_repairs_per_s_eil51"] = cnt / (time.perf_counter() - t0)
    # device-resident ALNS (vrp_alns_iterate): whole iterations (destroy, repair,
    # exact scoring, SA) per second, 1184 workers = 8 per SM, local search off
    from paper_2602_23685_b200 import alns as A
    init = A.construct_initial(inst)
    prm = A.AlnsParams(max_iter=100, pickup_reposition_interval=10**9, cross_agent_interval=10**9)
    ws = [A._Worker(inst, prm, A.worker_seed(3, i), init, None, None, i) for i in range(1184)]
    dw = A._DeviceWorkers(inst, prm, ws)
    dw.run(1, 5)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dw.run(6, 100)
    torch.cuda.synchronize()
    out["alns_iterations_per_s_eil51_1184_workers"] = 1184 * 95 / (time.perf_counter() - t0)
    # K1 on the other benchmark configs (decoded candidates, device-resident)
    for key in ("eil51", "kroA100", "a280"):
        ki = config_instance(key)
        # 2^20 candidates: larger than L2 at every n.  At eil51 the rate is
        # bimodal (~360 M or ~630 M evals/s) with where the op buffer lands in
        # device memory (scripts/probe_k1_bench_ctx.py); dsj1000 is not
        cnt = 1 << 20
        kops = torch.empty((cnt, 2 * ki.n), dtype=torch.int16, device=device)
        klens = torch.empty((cnt, ki.m), dtype=torch.int32, device=device)
        kg = torch.Generator(device=device).manual_seed(11)
        for s0 in range(0, cnt, 1 << 16):
            gg = torch.rand((1 << 16, 4 * ki.n), dtype=torch.float64, device=device, generator=kg)
            D.decode_batch(ki, gg, out={"ops": kops[s0:s0 + (1 << 16)], "lens": klens[s0:s0 + (1 << 16)]})
        res = {}
        for _ in range(2):
            D.makespan_batch(ki, kops, klens, mode=0, out=res)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            D.makespan_batch(ki, kops, klens, mode=0, out=res)
        e1.record()
        torch.cuda.synchronize()
        out[f"k1_evals_per_s_{key}"] = 5 * cnt / (e0.elapsed_time(e1) / 1e3)
        del kops, klens
    if pipeline_seconds > 0:
        # BASELINE's "best makespan at fixed time": the whole ALNS -> BRKGA
        # pipeline (pipeline.run_pipeline_budget) on the kroA100 pipeline config
        from paper_2602_23685_b200.pipeline import run_pipeline_budget
        kro = config_instance("kroA100")
        _, zb, tr = run_pipeline_budget(kro, seconds=pipeline_seconds)
        out[f"best_makespan_kroA100_{pipeline_seconds:g}s"] = zb
        out["initial_makespan_kroA100"] = tr[0][1]
        # and on the n = 999 config with the 60 s budget of BASELINE config 5
        # (the reference does not finish construct_initial in 60 s there)
        _, zb, tr = run_pipeline_budget(dsj, seconds=2 * pipeline_seconds)
        out[f"best_makespan_dsj1000_{2 * pipeline_seconds:g}s"] = zb
        out["initial_makespan_dsj1000"] = tr[0][1]
        # the same budget with the ALNS stage on at n = 999 (team-repair ALNS,
        # 148 workers after a shorter polish): the paper's ALNS -> BRKGA order
        _, zb, tr = run_pipeline_budget(dsj, seconds=2 * pipeline_seconds, alns_max_n=10**9, pool_size=148,
                                        alns_share=0.9, polish_share=0.3, final_share=0.3)
        out[f"best_makespan_dsj1000_{2 * pipeline_seconds:g}s_alns_on"] = zb
    return {k: round(v, 2) for k, v in out.items()}


def l2_gather_ceiling():
    """Measured random 4-byte gather rate of L2 (scripts/probes/l2gather.cu on
    a B200 of this pool, profiles/r02_l2gather.json): the best rate over the
    L2-resident table sizes (4-64 MB), G gathers/s."""
    p = REPO / "profiles" / "r02_l2gather.json"
    if not p.exists():
        return None
    rows = json.loads(p.read_text())["rows"]
    return max(max(r["ggather_s"].values()) for r in rows if r["table_bytes"] <= (64 << 20))


def k1_roofline(n, m, n_cand, ms_per_step, clocks):
    """Roofline of K1 (the timed kernel) against three ceilings, per GPU:
      issue     warp instructions per eval (ncu, profiles/k1_profile.json) x
                evals/s vs 148 SMs x 4 schedulers x SM clock (measured median
                under load) -- the binding ceiling of a dependent scalar replay;
      l2_gather the 2n + m leg gathers d[prev][c] per eval (4 B each, random,
                L2-resident int32 twin) vs the measured L2 gather ceiling;
      hbm       ncu DRAM bytes per eval x evals/s vs the measured HBM copy peak.
    The headline object is the ceiling with the largest fraction; the
    algorithmic-bytes figure of SURVEY §8(d) (32n + 12m + 12 B/eval) is kept
    beside it."""
    evals_s = n_cand / (ms_per_step / 1e3)
    hbm_peak, peak_kind = measured_peaks()
    prof = {}
    pp = REPO / "profiles" / "k1_profile.json"
    if pp.exists():
        prof = json.loads(pp.read_text())
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    per_eval_alg = algorithmic_bytes_per_eval(n, m)
    views = {}
    if prof.get("warp_inst_per_eval"):
        ach = prof["warp_inst_per_eval"] * evals_s / 1e9
        pk = 148 * 4 * sm_mhz / 1e3
        views["issue"] = {"achieved": round(ach, 1), "peak": round(pk, 1), "unit": "G warp-inst/s",
                          "frac": round(ach / pk, 4), "per_eval": prof["warp_inst_per_eval"],
                          "source": prof.get("source")}
    l2 = l2_gather_ceiling()
    if l2:
        g = 2 * n + m
        ach = g * evals_s / 1e9
        views["l2_gather"] = {"achieved": round(ach, 1), "peak": round(l2, 1), "unit": "G gathers/s",
                              "frac": round(ach / l2, 4), "per_eval": g,
                              "source": "profiles/r02_l2gather.json (scripts/probes/l2gather.cu)"}
    dram = prof.get("dram_bytes_per_eval")
    if dram:
        ach = dram * evals_s / 1e9
        views["hbm"] = {"achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(ach / hbm_peak, 4), "per_eval": dram, "peak_kind": peak_kind}
    alg = per_eval_alg * evals_s / 1e9
    bound = max(views, key=lambda k: views[k]["frac"]) if views else None
    head = views.get(bound) if bound else {"achieved": round(alg, 1), "peak": hbm_peak, "unit": "GB/s",
                                            "frac": round(alg / hbm_peak, 4)}
    return {"bound": bound or "hbm", "achieved": head["achieved"], "peak": head["peak"],
            "unit": head["unit"], "frac": head["frac"],
            "traffic": round(dram * n_cand) if dram else None,
            "traffic_source": "profiles/k1_profile.json: ncu dram__bytes_read+write per eval x candidates per launch",
            "ceilings": views,
            "algorithmic": {"bytes_per_eval": per_eval_alg, "achieved": round(alg, 1), "unit": "GB/s",
                            "peak": hbm_peak, "frac": round(alg / hbm_peak, 4),
                            "note": "SURVEY §8(d) bytes incl. L2-resident d/p gathers"},
            "sm_mhz_used": sm_mhz}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baselines(seconds: float = 6.0):
    """The reference algorithms of the secondary rates, timed on this box's
    host cores with the CPU oracle (C restatements of brkga.decode,
    brkga.evolve and insertion.reinsert_all; kind "port"), each on a bounded
    sample -- next to the GPU's decodes/s, generations/s and repairs/s."""
    from concurrent.futures import ThreadPoolExecutor
    import inputs as I
    from oracle import oracle as O
    from paper_2602_23685_b200.configs import config_instance
    threads = O.default_threads()
    out = {"cpu_model": cpu_model(), "cores": threads, "kind": "port"}
    dsj = config_instance("dsj1000")
    genes = I.chromosomes(dsj.n, 512, (136, 6001))
    t0, done = time.perf_counter(), 0
    while time.perf_counter() - t0 < seconds:
        O.decode_batch(dsj, genes, threads=threads)
        done += genes.shape[0]
    out["decodes_per_s_dsj1000_random"] = round(done / (time.perf_counter() - t0), 2)
    # evolve (numpy-Philox draws + [elite | mutant | offspring] build), one thread,
    # paper population N_p = 30,000 at a280 (4n = 1116 genes)
    a280 = config_instance("a280")
    pop = I.chromosomes(a280.n, 30000, (136, 6002))
    fit = np.random.default_rng(3).random(30000)
    g = I.philox(136, 6003)
    t0, gens = time.perf_counter(), 0
    while time.perf_counter() - t0 < seconds / 2 or gens == 0:
        pop = O.evolve(pop, fit, 0.15, 0.15, 0.7, g)
        gens += 1
    out["evolve_per_s_a280_Np30000_1thread"] = round(gens / (time.perf_counter() - t0), 3)
    # reinsert_all at eil51 (q = 5 picked, cascade included), instances over threads
    eil = config_instance("eil51")
    dec = O.decode_batch(eil, I.chromosomes(eil.n, 256, (7, 7)))
    cases = []
    for i in range(256):
        pick = I.philox(8, i).choice(np.arange(1, eil.n + 1), size=5, replace=False)
        o, l, r = O.remove_customers(eil, dec["ops"][i], dec["lens"][i], pick)
        cases.append((o[:2 * eil.n], l, r, (0, 2, 3, eil.m)[i % 4], i))

    def one(c):
        return O.reinsert_all(eil, c[0], c[1], c[2], c[3], I.philox(9, c[4]))[0]
    t0, done = time.perf_counter(), 0
    with ThreadPoolExecutor(threads) as ex:
        while time.perf_counter() - t0 < seconds:
            list(ex.map(one, cases))
            done += len(cases)
    out["alns_repairs_per_s_eil51"] = round(done / (time.perf_counter() - t0), 2)
    return out


def extra_distributed(dev, world, pipeline_seconds):
    """Legs that run at every N (BASELINE configs 4 and 5): the a280 BRKGA
    island model (N_p = 30,000 split over the ranks, ring migration of 32
    elites every 10 generations, incumbent min-all-reduce) -- global
    generations/s and the time of one migration + sync; and the dsj1000
    time-budgeted pipeline on every rank with a final min-all-reduce of the
    incumbent.  Times are max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2602_23685_b200 import brkga as B
    from paper_2602_23685_b200 import islands as IS
    from paper_2602_23685_b200 import rng as R
    from paper_2602_23685_b200.configs import config_instance
    rank = dist.get_rank() if world > 1 else 0

    def tmax(x):
        if world < 2:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    out = {}
    a280 = config_instance("a280")
    size = 30000 // world
    prm = B.BrkgaParams(population=size, generations=1)
    gen = R.philox_generator(5, R.BRKGA_STREAM + rank)
    eng = IS.DeviceIslandEngine(a280, prm, gen.random((size, 4 * a280.n)), gen)
    for _ in range(2):
        eng.generation()
    G, gen_s, mig_s = 20, 0.0, 0.0
    for g in range(1, G + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.generation()
        torch.cuda.synchronize()
        gen_s += time.perf_counter() - t0
        if g % 10 == 0:
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            IS.migrate(eng, 32)
            best, _, _ = IS.sync_incumbent(eng)
            torch.cuda.synchronize()
            mig_s += time.perf_counter() - t0
    gen_s, mig_s = tmax(gen_s), tmax(mig_s)
    out["islands_a280_generations_per_s_global_Np30000"] = round(G / gen_s, 2)
    out["islands_a280_migration_plus_sync_ms"] = round(1e3 * mig_s / (G // 10), 3)
    out["islands_a280_best_fitness"] = best
    if pipeline_seconds > 0 and world > 1:
        from paper_2602_23685_b200.pipeline import run_pipeline_budget_distributed
        dsj = config_instance("dsj1000")
        secs = 2 * pipeline_seconds
        _, zb, tr = run_pipeline_budget_distributed(dsj, seconds=secs)
        out[f"best_makespan_dsj1000_{secs:g}s_{world}gpu"] = zb
        out["initial_makespan_dsj1000"] = tr[0][1]
    return out


def workload_config(n, m, k, n_cand, world):
    """The `config` object both arms print (the driver compares them)."""
    return {"workload": f"{CONFIG}-derived 1R20 (n=999, m=6, k=4): exact_makespan of {n_cand} "
                        f"random-chromosome-decoded candidates per GPU per step",
            "n": n, "m": m, "k": k, "candidates_per_gpu": n_cand, "op_format": "int16",
            "l2": "inputs larger than L2 "
                  f"({n_cand * 2 * n * 2 / 1e9:.1f} GB ops per GPU), no flush",
            "parallelism": f"candidate sharding x{world}"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import inputs as I
    from oracle import oracle as O
    from paper_2602_23685_b200.configs import config_instance
    inst = config_instance(CONFIG)
    threads = O.default_threads()
    genes = I.chromosomes(inst.n, 2048, (136, 5000))
    dec = O.decode_batch(inst, genes, threads=threads)
    ops, lens = dec["ops"], dec["lens"]
    for _ in range(args.warmup):
        O.makespan_batch(inst, ops[:256], lens[:256], mode="exact", threads=threads)
    rates = []
    for _ in range(args.steps):
        r, _, _ = cpu_reference_rate(inst, ops, lens, threads, min_seconds=0.5)
        rates.append(r)
    value = float(statistics.median(rates))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * ops.shape[0] / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(inst.n, inst.m, inst.k, args.candidates, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"bounded sample of the workload: {ops.shape[0]} oracle-decoded "
                                       f"dsj1000 candidates re-scored for >=0.5 s per step (the rate, "
                                       f"evals/s, is per-candidate work independent of the batch size), "
                                       f"{threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2602_23685_b200 import device as D
    from paper_2602_23685_b200.configs import config_instance

    rank, world, local = dist_env()
    # VRP_BENCH_SHARE_GPU=1 (code-path test only): ranks share the visible
    # GPUs round-robin over gloo -- never used for a reported number
    shared = os.environ.get("VRP_BENCH_SHARE_GPU") == "1"
    if shared:
        local = local % torch.cuda.device_count()
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    inst = config_instance(CONFIG)
    n, m = inst.n, inst.m
    n_cand = args.candidates

    t_setup = time.perf_counter()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record()
    ops, lens, z_dec = make_candidates(inst, n_cand, seed=1000 + rank, device=dev)
    d1.record()
    torch.cuda.synchronize()
    decode_ms = d0.elapsed_time(d1)
    setup_s = time.perf_counter() - t_setup

    stream = torch.cuda.current_stream()
    out = {}
    D.makespan_batch(inst, ops, lens, mode=0, out=out)
    torch.cuda.synchronize()
    # sanity: K1 must reproduce the decoder's makespans
    if not args.no_verify and not (bool((out["status"] == 0).all()) and torch.equal(out["z"], z_dec)):
        raise SystemExit("bench: K1 disagrees with the decoder's makespans")

    for _ in range(args.warmup):
        D.makespan_batch(inst, ops, lens, mode=0, out=out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            D.makespan_batch(inst, ops, lens, mode=0, out=out)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    # integral exact K1 = the narrow/compact pass + the 64-bit fix-up pass
    # (csrc/makespan.cu launch_narrow); non-integral instances launch one kernel
    launches_per_step = 2 if D.device_instance(inst).integral else 1
    total_units = n_cand * world
    value = total_units * args.steps / (ms / 1e3)

    # ---- end to end through the public API: pinned host ops -> GPU -> host z/status
    e2e = None
    if not args.no_e2e:
        ne = min(n_cand, args.e2e_candidates)
        h_ops = torch.empty((ne, 2 * n), dtype=torch.int16, pin_memory=True)
        h_lens = torch.empty((ne, m), dtype=torch.int32, pin_memory=True)
        h_ops.copy_(ops[:ne])
        h_lens.copy_(lens[:ne])
        from paper_2602_23685_b200.schedule import score_host_batch
        res = score_host_batch(inst, h_ops, h_lens)  # warm
        torch.cuda.synchronize()
        steps_e = max(3, args.steps // 4)
        for _ in range(2):
            score_host_batch(inst, h_ops, h_lens)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps_e):
            res = score_host_batch(inst, h_ops, h_lens)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        assert np.array_equal(res[0], z_dec[:ne].cpu().numpy())
        e2e = {"value": ne * world * steps_e / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(ne * (2 * n * 2 + m * 4)),
               "d2h_bytes_per_step": int(ne * (8 + 4)),
               "candidates_per_step": ne, "steps": steps_e,
               "path": "schedule.score_host_batch: pinned int16 ops, chunked H2D/K1/D2H on 2 streams"}

    line = None
    if rank == 0:
        roof = k1_roofline(n, m, n_cand, ms_per_step, clk.summary())
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            import inputs as I
            from oracle import oracle as O
            threads = O.default_threads()
            cnt = 2048
            h = ops[:cnt].to(torch.int32).cpu().numpy()
            hl = lens[:cnt].cpu().numpy()
            rate, done, el = cpu_reference_rate(inst, h, hl, threads, min_seconds=args.cpu_seconds)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"{done} exact_makespan evals ({cnt} distinct decoded dsj1000 "
                             f"candidates, repeated) in {el:.1f} s on {threads} threads"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": workload_config(n, m, inst.k, n_cand, world),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
                "setup_s": round(setup_s, 2)}
        if not args.no_extra and world == 1:
            line["extra"] = extra_rates(dev, ops, lens, decode_ms, n_cand, args.pipeline_seconds)
            line["extra_cpu_baselines"] = cpu_baselines()
    if not args.no_extra:
        del ops, lens
        torch.cuda.empty_cache()
        dist_extra = extra_distributed(dev, world, args.pipeline_seconds)
        if rank == 0:
            line.setdefault("extra", {}).update(dist_extra)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N local ranks (one per GPU, NCCL), so the
    driver's plain invocation measures N GPUs.  Refuses when fewer than N GPUs
    are visible (VRP_BENCH_SHARE_GPU=1: code-path test, ranks share GPUs)."""
    import socket
    import subprocess
    if os.environ.get("VRP_BENCH_SHARE_GPU") != "1":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench: --gpus {n} but only {have} GPU(s) visible", file=sys.stderr)
            return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--candidates", type=int, default=1 << 20)
    ap.add_argument("--e2e-candidates", type=int, default=1 << 18)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--pipeline-seconds", type=float, default=30.0,
                    help="wall-clock budget of the best-makespan pipeline extra (0 = skip)")
    ap.add_argument("--no-verify", action="store_true", help="skip the K1 == decoder check (ablation builds)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
