"""Per-iteration cost of the lockstep batched ALNS (run_pool) at scale."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_23685_b200 import alns as A
from paper_2602_23685_b200.configs import config_instance
for key, W, iters in (("eil51", 64, 5), ("eil51", 512, 3), ("kroA100", 256, 3)):
    inst = config_instance(key)
    init = A.construct_initial(inst, 0) if key != "dsj1000" else None
    params = A.AlnsParams(max_iter=iters)
    t0 = time.perf_counter()
    workers = [A._Worker(inst, params, A.worker_seed(1, i), init, None, None, i) for i in range(W)]
    t1 = time.perf_counter()
    tp = tr = tc = 0.0
    for it in range(1, iters + 1):
        a = time.perf_counter()
        for w in workers:
            w.propose(it)
        b = time.perf_counter()
        res = A._repair_many(inst, workers)
        c = time.perf_counter()
        for w, (cand, z, failed) in zip(workers, res):
            w.conclude(it, cand, z, failed)
        d = time.perf_counter()
        tp += b - a; tr += c - b; tc += d - c
    print(f"{key} W={W}: init {t1-t0:.2f}s; per iteration: destroy(host) {tp/iters*1e3:.1f} ms, "
          f"repair+score(device) {tr/iters*1e3:.1f} ms, conclude {tc/iters*1e3:.1f} ms", flush=True)
