"""Best makespan at 60 s on the dsj1000 config for a few ALNS shares."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs  # noqa: E402
from paper_2602_23685_b200.pipeline import run_pipeline_budget  # noqa: E402
inst = configs.config_instance(sys.argv[1] if len(sys.argv) > 1 else "dsj1000")
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 60
for share, pool in ((0.8, 296),):
    t = time.perf_counter()
    sol, z, trace = run_pipeline_budget(inst, seconds=secs, alns_share=share, pool_size=pool)
    torch.cuda.synchronize()
    print(f"share={share} pool={pool}: best={z:.0f} in {time.perf_counter() - t:.1f}s "
          f"[{' '.join(f'{a:.0f}s:{b:.0f}' for a, b in trace[-6:])}]", flush=True)
