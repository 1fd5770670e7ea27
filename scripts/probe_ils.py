"""Timing of the pipeline's kick-and-polish rounds: python scripts/probe_ils.py KEY SECONDS"""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import alns as A, baselines as BL, configs, pipeline as P  # noqa: E402
from paper_2602_23685_b200.schedule import evaluate  # noqa: E402
key, secs = sys.argv[1], float(sys.argv[2])
inst = configs.config_instance(key)
sol = BL.two_opt_improve(inst, A.construct_initial(inst), move_budget=10**15, resume=True)
print("start", evaluate(inst, sol).makespan, flush=True)
t = time.perf_counter()
orig = BL.two_opt_improve


def timed(*a, **k):
    t1 = time.perf_counter()
    r = orig(*a, **k)
    print(f"  polish {time.perf_counter() - t1:.2f}s", flush=True)
    return r


BL.two_opt_improve = timed
last = time.perf_counter()
kick = P._Kicker(inst, sol, 0)
while time.perf_counter() + 1.2 * kick.last_s < t + secs - 0.5:
    s = kick.round(t + secs)
    if s is not None:
        print(f"improved {evaluate(inst, s).makespan:.0f} at {time.perf_counter() - t:.1f}s", flush=True)
print(f"ILS ended at {time.perf_counter() - t:.1f}s (deadline {secs}s)", flush=True)
