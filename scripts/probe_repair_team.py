"""K5 / device-ALNS timing at a280 and dsj1000: the team repair (a CTA per
instance, csrc/repair_team.cuh) against the warp-per-instance path.

    python scripts/probe_repair_team.py            # the in-tree library
    VRP_LIB=variants/libnoteam.so python scripts/probe_repair_team.py
Prints repairs/s for the dsj1000 parity cases and ALNS seconds per iteration
per worker (local search off)."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "tests/golden")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs as I  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_23685_b200 import alns as A  # noqa: E402
from paper_2602_23685_b200 import insertion as INS  # noqa: E402
from paper_2602_23685_b200.configs import config_instance  # noqa: E402


def repairs(key, count, q):
    inst = config_instance(key)
    dec = O.decode_batch(inst, I.chromosomes(inst.n, count, (81, 5)))
    parts, plens, rem = [], [], []
    for i in range(count):
        pick = I.philox(82, 5, i).choice(np.arange(1, inst.n + 1), size=q, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
    parts, plens = np.stack(parts), np.stack(plens)
    rks = [(0, 2, 3, inst.m)[i % 4] for i in range(count)]
    # warm-up at the full batch size (the first call of a size grows the scratch pool)
    INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(83, i) for i in range(count)])
    torch.cuda.synchronize()
    t = time.perf_counter()
    o, l, st = INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(83, i) for i in range(count)])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    sizes = [len(r) for r in rem]
    ok = True
    for i in range(min(count, 4)):
        g = I.philox(83, i)
        rst, ro, rl = O.reinsert_all(inst, parts[i], plens[i], rem[i], rks[i], g)
        ok &= bool(st[i] == rst and (rst or (np.array_equal(o[i], ro) and np.array_equal(l[i], rl))))
    print(f"repair {key:8s} N={count:4d} q={q:3d} removed mean {np.mean(sizes):6.1f} max {max(sizes):4d}: "
          f"{dt:7.3f} s  {count / dt:9.1f} repairs/s  oracle-equal(first 4)={ok}", flush=True)


def alns(key, W, iters):
    inst = config_instance(key)
    init = A.construct_initial(inst)
    params = A.AlnsParams(max_iter=iters, pickup_reposition_interval=10**9, cross_agent_interval=10**9)
    workers = [A._Worker(inst, params, A.worker_seed(1, i), init, None, None, i) for i in range(W)]
    dw = A._DeviceWorkers(inst, params, workers)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dw.drive()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    best = min(w.z_best for w in workers)
    print(f"alns   {key:8s} W={W:4d} iters={iters:4d}: {dt:8.2f} s  {dt / iters:8.3f} s/iter/worker-stretch  "
          f"{W * iters / dt:9.1f} it/s  z0={workers[0].stats.initial_makespan:.0f} best={best:.0f}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["repair", "alns"]
    if "repair" in what:
        repairs("a280", 64, 14)
        repairs("dsj1000", 16, 24)
        repairs("dsj1000", 148, 24)
    if "alns" in what:
        alns("a280", 148, 20)
        alns("dsj1000", 8, 3)
        alns("dsj1000", 148, 3)
