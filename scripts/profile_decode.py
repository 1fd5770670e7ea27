"""One K3 decode launch at dsj1000 for ncu: python scripts/profile_decode.py N"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs, device as D  # noqa: E402
inst = configs.config_instance("dsj1000")
N = int(sys.argv[1])
g = torch.rand((N, 4 * inst.n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
D.decode_batch(inst, g, want_solution=False)
torch.cuda.synchronize()
