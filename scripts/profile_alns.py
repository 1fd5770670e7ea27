"""One vrp_alns_iterate stretch for ncu: python scripts/profile_alns.py KEY W ITERS"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2602_23685_b200 import alns as A  # noqa: E402
from paper_2602_23685_b200 import configs  # noqa: E402

key, W, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = configs.config_instance(key)
init = A.construct_initial(inst)
params = A.AlnsParams(max_iter=iters, pickup_reposition_interval=10**9, cross_agent_interval=10**9)
workers = [A._Worker(inst, params, A.worker_seed(1, i), init, None, None, i) for i in range(W)]
dw = A._DeviceWorkers(inst, params, workers)
torch.cuda.synchronize()
t = time.perf_counter()
dw.run(1, iters)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"{key} W={W} iters={iters}: {dt:.3f}s  {W * iters / dt:.0f} it/s", flush=True)
