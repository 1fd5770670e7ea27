"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/golden.npz     -- inputs (small) and reference outputs
  tests/golden/golden.json    -- metadata: versions, per-config instance hashes
  paper_2602_23685_b200/data/gr17_base.json -- the reference's parse of pkg/data/gr17.tsp

Reference functions exercised (paths relative to pkg/src/vrp_rpd/):
  instance.parse_tsplib / build_instance   instance.py:200-401
  schedule.exact_makespan                  schedule.py:265-316
  schedule.evaluate                        schedule.py:188-257
  schedule.two_pass_estimate               schedule.py:345-393
  brkga.decode / encode                    brkga.py:92-222
  brkga.evolve (Generator(Philox) injected) brkga.py:231-252
"""
from __future__ import annotations

import json
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")
REF_DATA = Path("/root/reference/pkg/data")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

import vrp_rpd  # noqa: E402  (the reference)
from vrp_rpd import brkga as R_brkga  # noqa: E402
from vrp_rpd import instance as R_inst  # noqa: E402
from vrp_rpd import schedule as R_sched  # noqa: E402

import inputs as I  # noqa: E402
from paper_2602_23685_b200 import configs as C  # noqa: E402
from paper_2602_23685_b200 import instance as mine  # noqa: E402

STATUS = {None: 0, "CapacityViolation": 1, "Deadlock": 2, "MalformedSolution": 3}
CFG_ID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}
# (decode chromosomes, random candidates, block candidates)
COUNTS = {"gr17": (256, 256, 64), "eil51": (96, 128, 32), "kroA100": (48, 64, 16),
          "a280": (16, 32, 8), "dsj1000": (8, 16, 4)}


def ref_instance(key):
    spec = C.CONFIGS[key]
    if spec.edge_type == "EXPLICIT":
        raw = R_inst.load_tsplib_file(REF_DATA / "gr17.tsp")
    else:
        raw = R_inst.parse_tsplib(C.synthetic_tsplib(spec))
    return R_inst.build_instance(raw, R_inst.VariantSpec(spec.variant, C.VARIANT_SEED, 0))


def to_solution(ops_row, lens_row):
    return R_sched.Solution.from_lists(
        [[(c, R_sched.OpKind(k)) for c, k in t] for t in I.arrays_to_lists(ops_row, lens_row)])


def score(inst, ops, lens):
    """Reference exact_makespan / evaluate / two_pass on each candidate."""
    N = ops.shape[0]
    out = {k: np.zeros(N) for k in ("z_exact", "z_eval", "z_two")}
    out.update({k: np.zeros(N, np.int32) for k in ("st_exact", "st_eval", "st_two")})
    out["returns"] = np.zeros((N, inst.m))
    for i in range(N):
        sol = to_solution(ops[i], lens[i])
        for fn, tag in ((R_sched.exact_makespan, "exact"), (None, "eval"),
                        (R_sched.two_pass_estimate, "two")):
            try:
                if tag == "eval":
                    sch = R_sched.evaluate(inst, sol)
                    z = sch.makespan
                    out["returns"][i] = sch.returns
                else:
                    z = fn(inst, sol)
                st = 0
            except R_sched.ScheduleError as exc:
                z, st = 0.0, STATUS[type(exc).__name__]
            out[f"z_{tag}"][i] = z
            out[f"st_{tag}"][i] = st
    return out


def main():
    t0 = time.time()
    blob: dict = {}
    meta = {"python": platform.python_version(), "numpy": np.__version__,
            "reference": str(REF_SRC), "configs": {}}

    for key, spec in C.CONFIGS.items():
        cid = CFG_ID[key]
        n_dec, n_rand, n_blk = COUNTS[key]
        inst = ref_instance(key)
        d = np.array(inst.d, dtype=np.float64)
        p = np.array(inst.p, dtype=np.float64)
        n, m, k = inst.n, inst.m, inst.k
        if key == "gr17":
            inst.save(HERE.parent.parent / "paper_2602_23685_b200" / "data" / "gr17_base.json")
        # pin our own instance builder against the reference's
        ours = C.config_instance(key)
        od, op = ours.arrays()
        assert np.array_equal(od, d) and np.array_equal(op, p), key
        assert (ours.n, ours.m, ours.k) == (n, m, k), key
        meta["configs"][key] = {"n": n, "m": m, "k": k, "label": inst.label,
                                "d_sha": I.sha(d), "p_sha": I.sha(p),
                                "integral": bool(np.all(d == np.round(d)) and np.all(p == np.round(p)))}
        pre = f"{key}/"
        blob[pre + "p"] = p
        if n <= 100:
            blob[pre + "d"] = d

        # ---- decode: uniform chromosomes, encoded (tie-heavy) ones, strict mode
        genes = I.chromosomes(n, n_dec, (136, cid))
        params = R_brkga.BrkgaParams(population=max(20, n_dec))
        strict = R_brkga.BrkgaParams(population=max(20, n_dec), wait_relaxation=False)
        dec_ops = np.zeros((n_dec, 2 * n), np.int32)
        dec_lens = np.zeros((n_dec, m), np.int32)
        recs = {k2: [] for k2 in ("fitness", "makespan", "scheduled", "visits")}
        enc = []
        for i in range(n_dec):
            r = R_brkga.decode(genes[i], inst, params)
            o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in r.solution.tours], n)
            dec_ops[i], dec_lens[i] = o, l
            recs["fitness"].append(r.fitness)
            recs["makespan"].append(r.makespan)
            recs["scheduled"].append(r.scheduled_count)
            recs["visits"].append(r.op_visits)
            if i < max(2, n_dec // 8):
                enc.append(R_brkga.encode(inst, r.solution))
        blob[pre + "dec_genes_sha"] = np.frombuffer(I.sha(genes).encode(), np.uint8)
        blob[pre + "dec_ops"] = dec_ops
        blob[pre + "dec_lens"] = dec_lens
        for k2, v in recs.items():
            blob[pre + "dec_" + k2] = np.array(v)
        # encoded chromosomes (many exactly-equal keys) + strict-mode decodes
        enc = np.array(enc)
        blob[pre + "enc_genes"] = enc
        for tag, prm, src in (("enc", params, enc), ("strict", strict, genes[: len(enc)])):
            o_all = np.zeros((len(src), 2 * n), np.int32)
            l_all = np.zeros((len(src), m), np.int32)
            fit, mk, sc, vi = [], [], [], []
            for i in range(len(src)):
                r = R_brkga.decode(src[i], inst, prm)
                o_all[i], l_all[i] = I.lists_to_arrays(
                    [[(c, kd.value) for c, kd in t] for t in r.solution.tours], n)
                fit.append(r.fitness); mk.append(r.makespan)
                sc.append(r.scheduled_count); vi.append(r.op_visits)
            blob[pre + f"{tag}_ops"] = o_all
            blob[pre + f"{tag}_lens"] = l_all
            blob[pre + f"{tag}_fitness"] = np.array(fit)
            blob[pre + f"{tag}_makespan"] = np.array(mk)
            blob[pre + f"{tag}_scheduled"] = np.array(sc)
            blob[pre + f"{tag}_visits"] = np.array(vi)

        # ---- makespan family on decoded / random / block / perturbed candidates
        rnd_ops, rnd_lens = I.random_candidates(n, m, n_rand, (136, cid, 1))
        blk_ops, blk_lens = I.block_candidates(n, m, k, n_blk, (136, cid, 2))
        swp_ops = I.swap_perturb(dec_ops, dec_lens, (136, cid, 3))
        # malformed: duplicate one op in a few decoded candidates
        mal_ops = dec_ops[: min(4, n_dec)].copy()
        if n > 1:
            mal_ops[:, 1] = mal_ops[:, 0]
        sets = {"dec": (dec_ops, dec_lens), "rnd": (rnd_ops, rnd_lens),
                "blk": (blk_ops, blk_lens), "swp": (swp_ops, dec_lens),
                "mal": (mal_ops, dec_lens[: len(mal_ops)])}
        for tag, (o, l) in sets.items():
            if tag != "dec":
                blob[pre + f"{tag}_ops"] = o
                blob[pre + f"{tag}_lens"] = l
            res = score(inst, o, l)
            for k2, v in res.items():
                blob[pre + f"{tag}_{k2}"] = v
        print(f"{key}: n={n} m={m} k={k} done at {time.time() - t0:.1f}s", flush=True)

    # ---- evolve with an injected Generator(Philox)
    ev = []
    for j, (N, G, frac_e, frac_m, bias, tie) in enumerate([
            (20, 8, 0.15, 0.15, 0.7, False), (60, 64, 0.15, 0.15, 0.7, True),
            (200, 200, 0.15, 0.15, 0.7, True), (257, 120, 0.2, 0.1, 0.6, False),
            (10, 6, 0.15, 0.15, 1.0, False), (1000, 32, 0.15, 0.15, 0.7, True)]):
        g = I.philox(7, j)
        pop = g.random((N, G))
        fit = g.random(N)
        if tie:
            fit = np.round(fit * 7.0)
        rng = I.philox(11, j)
        prm = R_brkga.BrkgaParams(population=N, elite_fraction=frac_e,
                                  mutant_fraction=frac_m, elite_bias=bias)
        out = R_brkga.evolve(pop, fit, prm, rng)
        st = rng.bit_generator.state
        blob[f"evolve/{j}/out"] = out
        ev.append({"N": N, "G": G, "elite": frac_e, "mutant": frac_m, "bias": bias,
                   "tie": tie, "pop_key": [7, j], "rng_key": [11, j],
                   "final_counter": [int(x) for x in st["state"]["counter"]],
                   "final_buffer_pos": int(st["buffer_pos"]),
                   "final_has_uint32": int(st["has_uint32"]),
                   "final_uinteger": int(st["uinteger"])})
    meta["evolve"] = ev

    # ---- warm start constructors, encode, warm_start_population (brkga.py:260-424)
    for key in C.CONFIGS:
        inst = ref_instance(key)
        pre = f"{key}/"
        for tag, fn in (("greedy", R_brkga._greedy_ops_solution),
                        ("lb", R_brkga._load_balanced_solution), ("spt", R_brkga._spt_solution)):
            sol = fn(inst)
            o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in sol.tours], inst.n)
            blob[pre + f"ws_{tag}_ops"], blob[pre + f"ws_{tag}_lens"] = o, l
            blob[pre + f"ws_{tag}_enc"] = R_brkga.encode(inst, sol)
        if inst.n <= 300:
            inc = to_solution(blob[pre + "dec_ops"][0], blob[pre + "dec_lens"][0])
            prm = R_brkga.BrkgaParams(population=64, generations=3)
            pop = R_brkga.warm_start_population(inst, inc, prm, I.philox(13, CFG_ID[key]))
            blob[pre + "ws_pop"] = pop
        print(f"warm start {key} done at {time.time() - t0:.1f}s", flush=True)

    # ---- run_brkga driven by Generator(Philox(key=(seed, BRKGA_STREAM))) instead of
    # PCG64(seed): the reference's own loop, its generator swapped (rng.py)
    BRKGA_STREAM = 0xB4C6A
    runs = []
    insts = {key: ref_instance(key) for key in ("gr17", "eil51", "kroA100")}
    orig_pcg = np.random.PCG64
    try:
        np.random.PCG64 = lambda s: (np.random.Philox(key=(int(s), BRKGA_STREAM))
                                     if isinstance(s, (int, np.integer)) else orig_pcg(s))
        for j, (key, N_p, T, seed, warm) in enumerate([("gr17", 60, 8, 5, False), ("gr17", 40, 12, 9, True),
                                                       ("eil51", 50, 6, 3, False), ("kroA100", 30, 4, 11, True)]):
            inst = insts[key]
            prm = R_brkga.BrkgaParams(population=N_p, generations=T)
            wp = None
            if warm:
                inc = to_solution(blob[f"{key}/dec_ops"][0], blob[f"{key}/dec_lens"][0])
                wp = R_brkga.warm_start_population(inst, inc, prm, I.philox(17, j))
                blob[f"brkga/{j}/warm"] = wp
            best, stats = R_brkga.run_brkga(inst, prm, warm_population=wp, seed=seed)
            o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in best.tours], inst.n)
            blob[f"brkga/{j}/ops"], blob[f"brkga/{j}/lens"] = o, l
            blob[f"brkga/{j}/trace"] = np.array([f for _, f in stats.trace])
            runs.append({"key": key, "population": N_p, "generations": T, "seed": seed, "warm": warm,
                         "best_fitness": stats.best_fitness, "decodes": stats.decodes})
    finally:
        np.random.PCG64 = orig_pcg
    meta["brkga_runs"] = runs

    # ---- removal cascade + repair (insertion.py:379-516) and destroy (alns.py:182-251),
    # the reference driven by Generator(Philox) where it takes an rng
    from vrp_rpd import alns as R_alns
    from vrp_rpd import insertion as R_ins
    repairs, destroys = [], []
    for key, ncase, q in (("gr17", 12, 4), ("eil51", 12, 5), ("kroA100", 8, 5), ("a280", 4, 8)):
        inst = ref_instance(key)
        for j in range(ncase):
            sol = to_solution(blob[f"{key}/dec_ops"][j], blob[f"{key}/dec_lens"][j])
            pick = I.philox(31, CFG_ID[key], j).choice(np.arange(1, inst.n + 1), size=q, replace=False)
            tours, removed = R_ins.remove_customers(inst, sol, [int(x) for x in pick])
            po, pl = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in tours], inst.n)
            regret_k = (0, 2, 3, inst.m)[j % 4]
            use_rng = j % 6 != 5
            rng = I.philox(37, CFG_ID[key], j) if use_rng else None
            ctx = R_ins.InsertionContext(inst, tours)
            try:
                R_ins.reinsert_all(ctx, removed, regret_k=regret_k, rng=rng)
                st = 0
                ro, rl = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in ctx.tours], inst.n)
            except R_ins.RepairFailed:
                st, ro, rl = 1, np.full(2 * inst.n, -1, np.int32), np.zeros(inst.m, np.int32)
            tag = f"repair/{len(repairs)}"
            blob[tag + "/pick"] = np.asarray(pick, np.int32)
            blob[tag + "/partial_ops"], blob[tag + "/partial_lens"] = po, pl
            blob[tag + "/removed"] = np.asarray(removed, np.int32)
            blob[tag + "/ops"], blob[tag + "/lens"] = ro, rl
            rs = rng.bit_generator.state if use_rng else None
            repairs.append({"key": key, "case": j, "regret_k": regret_k, "rng": use_rng, "status": st,
                            "final_counter": [int(x) for x in rs["state"]["counter"]] if rs else None,
                            "final_buffer_pos": int(rs["buffer_pos"]) if rs else None,
                            "final_has_uint32": int(rs["has_uint32"]) if rs else None,
                            "final_uinteger": int(rs["uinteger"]) if rs else None})
        for j, op in enumerate(R_alns.DESTROY_OPERATORS * 2):
            sol = to_solution(blob[f"{key}/dec_ops"][j], blob[f"{key}/dec_lens"][j])
            rng = I.philox(41, CFG_ID[key], j)
            partial, removed = R_alns.destroy(inst, sol, op, q, rng)
            po, pl = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in partial.tours], inst.n)
            tag = f"destroy/{len(destroys)}"
            blob[tag + "/ops"], blob[tag + "/lens"] = po, pl
            blob[tag + "/removed"] = np.asarray(removed, np.int32)
            rs = rng.bit_generator.state
            destroys.append({"key": key, "case": j, "operator": op, "q": q,
                             "final_counter": [int(x) for x in rs["state"]["counter"]],
                             "final_buffer_pos": int(rs["buffer_pos"]),
                             "final_has_uint32": int(rs["has_uint32"]),
                             "final_uinteger": int(rs["uinteger"])})
        print(f"repair/destroy {key} done at {time.time() - t0:.1f}s", flush=True)
    meta["repairs"] = repairs
    meta["destroys"] = destroys

    # ---- construction + local search (alns.py:290-487) and whole ALNS runs
    # (alns.py:536-640) with _rng_for swapped to Generator(Philox(key=(seed, ALNS_STREAM)))
    ALNS_STREAM = 0xA1B5
    for key in ("gr17", "eil51", "kroA100"):
        inst = ref_instance(key)
        sol = R_alns.construct_initial(inst, seed=0)
        o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in sol.tours], inst.n)
        blob[f"ci/{key}/ops"], blob[f"ci/{key}/lens"] = o, l
        for j in range(3):
            base = to_solution(blob[f"{key}/dec_ops"][j], blob[f"{key}/dec_lens"][j])
            for tag, fn in (("pr", R_alns.pickup_repositioning), ("ca", R_alns.cross_agent_relocation)):
                out = fn(inst, base)
                o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in out.tours], inst.n)
                blob[f"ls/{key}/{tag}/{j}/ops"], blob[f"ls/{key}/{tag}/{j}/lens"] = o, l
        print(f"construct/LS {key} done at {time.time() - t0:.1f}s", flush=True)
    orig_rng_for = R_alns._rng_for
    runs = []
    try:
        R_alns._rng_for = lambda seed: np.random.Generator(np.random.Philox(key=(int(seed), ALNS_STREAM)))
        for j, (key, iters, seed, init, extra) in enumerate([
                ("gr17", 60, 3, None, {}), ("gr17", 240, 7, None, {"weight_interval": 50}),
                ("eil51", 30, 5, None, {}), ("kroA100", 8, 2, "dec", {}),
                ("eil51", 25, 9, "dec", {"stagnation_threshold": 5, "t0": 0.001})]):
            inst = ref_instance(key)
            prm = R_alns.AlnsParams(max_iter=iters, **extra)
            initial = to_solution(blob[f"{key}/dec_ops"][0], blob[f"{key}/dec_lens"][0]) if init else None
            best, st = R_alns.run_alns(inst, prm, seed=seed, initial=initial)
            o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in best.tours], inst.n)
            blob[f"alns/{j}/ops"], blob[f"alns/{j}/lens"] = o, l
            runs.append({"key": key, "iters": iters, "seed": seed, "init": init, "extra": extra,
                         "best_trace": st.best_trace, "accepted": st.accepted,
                         "rejected": st.rejected_candidates, "reheats": st.reheats,
                         "final_temperature": st.final_temperature, "attempts": st.attempts,
                         "initial_makespan": st.initial_makespan,
                         "weight_rows": st.weight_rows})
            print(f"alns run {j} done at {time.time() - t0:.1f}s", flush=True)
    finally:
        R_alns._rng_for = orig_rng_for
    meta["alns_runs"] = runs

    # ---- run_pipeline (bench.py:204-222), every PCG64 stream -> Philox
    from vrp_rpd import bench as R_bench
    pipes = []
    orig_pcg = np.random.PCG64
    try:
        R_alns._rng_for = lambda seed: np.random.Generator(np.random.Philox(key=(int(seed), ALNS_STREAM)))
        np.random.PCG64 = lambda s: (np.random.Philox(key=(int(s), BRKGA_STREAM))
                                     if isinstance(s, (int, np.integer)) else orig_pcg(s))
        for j, (key, iters, N_p, T, seed) in enumerate([("gr17", 40, 60, 5, 4), ("eil51", 12, 40, 3, 6)]):
            inst = insts.get(key) or ref_instance(key)
            sol, inc = R_bench.run_pipeline(inst, R_alns.AlnsParams(max_iter=iters),
                                            R_brkga.BrkgaParams(population=N_p, generations=T), seed)
            for tag, x in (("sol", sol), ("inc", inc)):
                o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in x.tours], inst.n)
                blob[f"pipe/{j}/{tag}_ops"], blob[f"pipe/{j}/{tag}_lens"] = o, l
            pipes.append({"key": key, "iters": iters, "population": N_p, "generations": T, "seed": seed})
    finally:
        R_alns._rng_for = orig_rng_for
        np.random.PCG64 = orig_pcg
    meta["pipelines"] = pipes

    # ---- heuristic polish two_opt_improve (baselines.py:372-455), deterministic
    from vrp_rpd import baselines as R_base
    polish = []
    for key, cases, budget in (("gr17", 3, None), ("eil51", 2, 1500), ("kroA100", 1, 400)):
        inst = insts.get(key) or ref_instance(key)
        for j in range(cases):
            sol = to_solution(blob[f"{key}/dec_ops"][j], blob[f"{key}/dec_lens"][j])
            out = R_base.two_opt_improve(inst, sol, move_budget=budget)
            o, l = I.lists_to_arrays([[(c, kd.value) for c, kd in t] for t in out.tours], inst.n)
            blob[f"polish/{len(polish)}/ops"], blob[f"polish/{len(polish)}/lens"] = o, l
            polish.append({"key": key, "case": j, "budget": budget})
    meta["polish"] = polish
    print(f"two_opt done at {time.time() - t0:.1f}s", flush=True)

    # ---- hint vehicle edge cases (brkga.py:82-89)
    genes = np.array([0.0, 1 / 3, 2 / 3, 1 / 6, 0.5, np.nextafter(1.0, 0), 0.999999999,
                      np.nextafter(1 / 3, 0), np.nextafter(2 / 3, 0), 0.2, 0.4, 0.6, 0.8])
    hv = np.array([[R_brkga._hint_vehicle(mm, float(x)) for x in genes] for mm in (1, 2, 3, 5, 6, 7)])
    blob["hint/genes"] = genes
    blob["hint/out"] = hv

    np.savez_compressed(HERE / "golden.npz", **blob)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1))
    print(f"wrote golden in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
