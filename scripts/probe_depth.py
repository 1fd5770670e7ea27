"""Lockstep depth per candidate vs its warp's (needs the _depth side build)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2602_23685_b200 import configs, device as D  # noqa: E402
inst = configs.config_instance("dsj1000")
N = 1 << 16
g = torch.rand((N, 4 * inst.n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
dec = D.decode_batch(inst, g, op_dtype=torch.int16)
r = D.makespan_batch(inst, dec["ops"], dec["lens"], mode=0, want_bottleneck=True)
b = r["bottleneck"].cpu().numpy()
mine, allw = b // 1000, b % 1000
print("candidate depth mean %.1f sd %.1f min %d max %d; warp depth mean %.1f; ratio %.3f"
      % (mine.mean(), mine.std(), mine.min(), mine.max(), allw.mean(), allw.mean() / mine.mean()))
