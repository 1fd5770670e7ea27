"""Best makespan at a fixed wall-clock budget (run_pipeline_budget):
python scripts/probe_pipeline.py KEY SECONDS"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2602_23685_b200 import configs  # noqa: E402
from paper_2602_23685_b200.pipeline import run_pipeline_budget  # noqa: E402

key, secs = sys.argv[1], float(sys.argv[2])
inst = configs.config_instance(key)
variants = [{}] + [dict(v) for v in ({"final_share": 0.95}, {"final_share": 0.5}, {"alns_max_n": 50})]
for kw in variants:
    t = time.perf_counter()
    sol, z, trace = run_pipeline_budget(inst, seconds=secs, **kw)
    torch.cuda.synchronize()
    pts = " ".join(f"{a:.0f}s:{b:.0f}" for a, b in trace[-6:])
    print(f"{key} {kw}: best={z:.0f} in {time.perf_counter() - t:.1f}s  [{pts}]", flush=True)
