"""Best makespan at a fixed wall-clock budget (run_pipeline_budget) for a few
pool sizes / ALNS shares.  python scripts/probe_pipeline.py KEY SECONDS"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2602_23685_b200 import configs  # noqa: E402
from paper_2602_23685_b200.pipeline import run_pipeline_budget  # noqa: E402

key, secs = sys.argv[1], float(sys.argv[2])
inst = configs.config_instance(key)
for pool, share, fit in ((148, 0.5, True), (296, 0.5, True), (1184, 0.5, True), (296, 0.8, True),
                         (296, 0.5, False)):
    t = time.perf_counter()
    sol, z, trace = run_pipeline_budget(inst, seconds=secs, alns_share=share, pool_size=pool, fit_cooling=fit)
    torch.cuda.synchronize()
    pts = " ".join(f"{a:.0f}s:{b:.0f}" for a, b in trace[:: max(1, len(trace) // 8)])
    print(f"{key} pool={pool:5d} share={share:.1f} fit={int(fit)}: best={z:.0f} in {time.perf_counter() - t:.1f}s  [{pts}]",
          flush=True)
