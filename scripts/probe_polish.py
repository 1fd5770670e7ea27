"""two_opt_improve as a time-boxed polish: python scripts/probe_polish.py KEY SECONDS..."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import alns as A, baselines as BL, configs  # noqa: E402
from paper_2602_23685_b200.schedule import evaluate  # noqa: E402
key = sys.argv[1]
inst = configs.config_instance(key)
sol = A.construct_initial(inst)
z0 = evaluate(inst, sol).makespan
for secs in map(float, sys.argv[2:]):
    for resume in (False, True):
        t1 = time.perf_counter()
        out = BL.two_opt_improve(inst, sol, move_budget=10**12, deadline=t1 + secs, resume=resume)
        torch.cuda.synchronize()
        print(f"{key}: initial {z0:.0f} -> polished {evaluate(inst, out).makespan:.0f} in "
              f"{time.perf_counter() - t1:.1f}s (deadline {secs}s, resume={resume})", flush=True)
