"""Best-so-far makespan of the REFERENCE pipeline (pure Python, one core)
under a wall-clock cap -- the CPU side of BASELINE's 'best makespan at fixed
time'.  The reference has no time budget, so this harness
wraps its exact_makespan / evaluate: every scored candidate updates the
best-so-far, and the run is stopped at the deadline.  Runs in the build
container only (needs /root/reference).

    python scripts/ref_budget.py KEY SECONDS
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests" / "golden"))
from make_golden import ref_instance  # noqa: E402
from vrp_rpd import alns as R_alns, bench as R_bench, brkga as R_brkga, schedule as R_s  # noqa: E402


class Deadline(Exception):
    pass


def main(key, secs):
    inst = ref_instance(key)
    t0 = time.perf_counter()
    state = {"best": float("inf"), "trace": []}
    orig_exact, orig_eval = R_s.exact_makespan, R_s.evaluate

    def note(z):
        el = time.perf_counter() - t0
        if z < state["best"]:
            state["best"] = z
            state["trace"].append((round(el, 2), z))
        if el > secs:
            raise Deadline()

    def exact(instance, sol):
        z = orig_exact(instance, sol)
        note(z)
        return z

    def evaluate(instance, sol):
        s = orig_eval(instance, sol)
        note(s.makespan)
        return s

    for mod in (R_alns, R_brkga, R_s, R_bench):
        if hasattr(mod, "exact_makespan"):
            mod.exact_makespan = exact
        if hasattr(mod, "evaluate"):
            mod.evaluate = evaluate
    try:
        R_bench.run_pipeline(inst, R_alns.AlnsParams(), R_brkga.BrkgaParams(), seed=0)
        done = True
    except Deadline:
        done = False
    print(json.dumps({"key": key, "seconds": secs, "finished": done, "best": state["best"],
                      "trace": state["trace"][-12:]}))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
