"""Quick throughput probe of K3 decode, BRKGA generations and K5 repair (GPU)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests" / "golden"))
import inputs as I  # noqa: E402
from paper_2602_23685_b200 import brkga as B  # noqa: E402
from paper_2602_23685_b200 import device as D  # noqa: E402
from paper_2602_23685_b200 import insertion as INS  # noqa: E402
from paper_2602_23685_b200.configs import config_instance  # noqa: E402


def cuda_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


for key in ("gr17", "eil51", "kroA100", "a280", "dsj1000"):
    inst = config_instance(key)
    N = 30000
    genes = torch.rand((N, 4 * inst.n), dtype=torch.float64, device="cuda")
    out = {}
    t = cuda_time(lambda: D.decode_batch(inst, genes, want_solution=False, out=out))
    print(f"decode {key}: {N / t:,.0f} chrom/s (random chromosomes, N={N})", flush=True)
    params = B.BrkgaParams(population=N, generations=3)
    t0 = time.perf_counter()
    B.run_brkga(inst, params, seed=1)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print(f"run_brkga {key}: N_p={N}, 3 gens in {el:.3f}s -> {3 / el:.2f} gen/s (incl. gen-0 decode)", flush=True)

for key, q in (("eil51", 5), ("kroA100", 5), ("a280", 8)):
    inst = config_instance(key)
    cnt = 1024
    dec = D.decode_batch(inst, torch.rand((cnt, 4 * inst.n), dtype=torch.float64, device="cuda"))
    ops, lens = dec["ops"].cpu().numpy(), dec["lens"].cpu().numpy()
    from oracle import oracle as O
    parts, plens, rem = [], [], []
    for i in range(cnt):
        pick = I.philox(5, i).choice(np.arange(1, inst.n + 1), size=q, replace=False)
        o, l, r = O.remove_customers(inst, ops[i], lens[i], pick)
        parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
    parts, plens = np.stack(parts), np.stack(plens)
    gens = [I.philox(6, i) for i in range(cnt)]
    t0 = time.perf_counter()
    o, l, st = INS.reinsert_batch(inst, parts, plens, rem, [i % 4 and (0, 2, 3, 6)[i % 4] for i in range(cnt)], gens)
    el = time.perf_counter() - t0
    print(f"repair {key}: {cnt} instances (mean |removed| {np.mean([len(r) for r in rem]):.1f}) in {el:.3f}s "
          f"-> {cnt / el:,.0f} repairs/s, failed {int((st != 0).sum())}", flush=True)
