"""Small driver for ncu captures of K3 (decode, dsj1000) and K5 (repair, eil51)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests" / "golden"))
import inputs as I  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_23685_b200 import device as D  # noqa: E402
from paper_2602_23685_b200 import insertion as INS  # noqa: E402
from paper_2602_23685_b200.configs import config_instance  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("decode", "both"):
    inst = config_instance("dsj1000")
    genes = torch.rand((8192, 4 * inst.n), dtype=torch.float64, device="cuda")
    for _ in range(2):
        D.decode_batch(inst, genes, want_solution=False)
    torch.cuda.synchronize()
if which in ("repair", "both"):
    inst = config_instance("eil51")
    cnt = 1024
    dec = O.decode_batch(inst, I.chromosomes(inst.n, cnt, (7, 7)))
    parts, plens, rem = [], [], []
    for i in range(cnt):
        pick = I.philox(8, i).choice(np.arange(1, inst.n + 1), size=5, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
    for _ in range(2):
        INS.reinsert_batch(inst, np.stack(parts), np.stack(plens), rem,
                           [(0, 2, 3, 6)[i % 4] for i in range(cnt)], [I.philox(9, i) for i in range(cnt)])
    torch.cuda.synchronize()
print("ok")
