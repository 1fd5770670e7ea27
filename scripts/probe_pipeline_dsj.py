"""Best makespan at a fixed budget on the dsj1000 config: the budget
pipeline with ALNS off (alns_max_n gate) and on, for a few shares/pools.
    python scripts/probe_pipeline_dsj.py [seconds] [variant ...]"""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs  # noqa: E402
from paper_2602_23685_b200.pipeline import run_pipeline_budget  # noqa: E402

inst = configs.config_instance("dsj1000")
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60
VARIANTS = {
    "off": dict(alns_max_n=400),
    "on148": dict(alns_max_n=10**9, pool_size=148, alns_share=0.8),
    "on296": dict(alns_max_n=10**9, pool_size=296, alns_share=0.8),
    "on148_p30": dict(alns_max_n=10**9, pool_size=148, alns_share=0.9, polish_share=0.3, final_share=0.3),
}
for name in sys.argv[2:] or ["off", "on148"]:
    t = time.perf_counter()
    sol, z, trace = run_pipeline_budget(inst, seconds=secs, **VARIANTS[name])
    torch.cuda.synchronize()
    print(f"{name}: best={z:.0f} in {time.perf_counter() - t:.1f}s "
          f"[{' '.join(f'{a:.0f}s:{b:.0f}' for a, b in trace[-8:])}]", flush=True)
