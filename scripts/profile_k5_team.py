"""One K5 team launch (16 dsj1000 repairs, q = 24 picked + cascade) after a
warm-up, for ncu:  ncu -k regex:repair_team --set full -s 1 -c 1 python scripts/profile_k5_team.py"""
import sys

sys.path[:0] = [".", "tests", "tests/golden"]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs as I  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_23685_b200 import insertion as INS  # noqa: E402
from paper_2602_23685_b200.configs import config_instance  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 16
inst = config_instance("dsj1000")
dec = O.decode_batch(inst, I.chromosomes(inst.n, count, (81, 5)))
parts, plens, rem = [], [], []
for i in range(count):
    pick = I.philox(82, 5, i).choice(np.arange(1, inst.n + 1), size=24, replace=False)
    o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
    parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
parts, plens = np.stack(parts), np.stack(plens)
rks = [(0, 2, 3, inst.m)[i % 4] for i in range(count)]
for _ in range(2):
    INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(83, i) for i in range(count)])
torch.cuda.synchronize()
print("ok")
