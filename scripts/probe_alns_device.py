"""ALNS iterations/s of the device engine (vrp_alns_iterate) vs worker count.

    python scripts/probe_alns_device.py [key ...]
Kernel-only stretches (local search off) and the default cadence."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import torch  # noqa: E402

from paper_2602_23685_b200 import alns as A  # noqa: E402
from paper_2602_23685_b200 import configs  # noqa: E402


def probe(key, W, iters, ls):
    inst = configs.config_instance(key)
    init = A.construct_initial(inst)
    kw = {} if ls else {"pickup_reposition_interval": 10**9, "cross_agent_interval": 10**9}
    params = A.AlnsParams(max_iter=iters, **kw)
    workers = [A._Worker(inst, params, A.worker_seed(1, i), init, None, None, i) for i in range(W)]
    dw = A._DeviceWorkers(inst, params, workers)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dw.drive()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    best = min(w.z_best for w in workers)
    print(f"{key:8s} W={W:5d} iters={iters:5d} ls={int(ls)} {dt:7.2f}s  {W * iters / dt:10.0f} it/s "
          f"({dt / iters * 1e3:7.2f} ms/iter)  z0={workers[0].stats.initial_makespan:.0f} best={best:.0f}",
          flush=True)


if __name__ == "__main__":
    keys = sys.argv[1:] or ["eil51", "kroA100", "a280", "dsj1000"]
    plan = {"gr17": [(148, 400), (1184, 200)], "eil51": [(148, 400), (592, 200), (1184, 200)],
            "kroA100": [(148, 200), (592, 100), (1184, 100)], "a280": [(148, 60), (592, 40)],
            "dsj1000": [(148, 10), (296, 10)]}
    for key in keys:
        for W, it in plan[key]:
            probe(key, W, it, False)
        W, it = plan[key][0]
        probe(key, W, it, True)
