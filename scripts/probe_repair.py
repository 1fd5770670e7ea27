"""K5 repairs/s as in bench.py's extra, repeated: python scripts/probe_repair.py"""
import sys
import time
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import inputs as I  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_23685_b200 import insertion as INS  # noqa: E402
from paper_2602_23685_b200.configs import config_instance  # noqa: E402
inst = config_instance("eil51")
cnt = 1024
dec = O.decode_batch(inst, I.chromosomes(inst.n, cnt, (7, 7)))
parts, plens, rem = [], [], []
for i in range(cnt):
    pick = I.philox(8, i).choice(np.arange(1, inst.n + 1), size=5, replace=False)
    o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
    parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
parts, plens = np.stack(parts), np.stack(plens)
rks = [(0, 2, 3, inst.m)[i % 4] for i in range(cnt)]
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(9, i) for i in range(cnt)])
    torch.cuda.synchronize()
    print(f"rep {rep}: {cnt / (time.perf_counter() - t0):.0f} repairs/s", flush=True)
