"""Timing of construct_initial and the batched local search at scale."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2602_23685_b200 import alns as A  # noqa: E402
from paper_2602_23685_b200 import localsearch as LS  # noqa: E402
from paper_2602_23685_b200 import configs  # noqa: E402
from paper_2602_23685_b200.schedule import evaluate  # noqa: E402

for key in sys.argv[1:] or ["a280", "dsj1000"]:
    inst = configs.config_instance(key)
    t = time.perf_counter()
    sol = A.construct_initial(inst)
    torch.cuda.synchronize()
    print(f"{key}: construct_initial {time.perf_counter() - t:.2f}s z={evaluate(inst, sol).makespan:.0f}", flush=True)
    o, l = sol.to_arrays(inst.n)
    for name, fn in (("pickup", LS.pickup_repositioning_batch), ("cross", LS.cross_agent_relocation_batch)):
        t = time.perf_counter()
        _, _, z = fn(inst, o[None, :2 * inst.n], l[None])
        torch.cuda.synchronize()
        print(f"  {name} LS on the constructed solution: {time.perf_counter() - t:.2f}s z={z[0]:.0f}", flush=True)
