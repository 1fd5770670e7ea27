import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_23685_b200 import device as D
from paper_2602_23685_b200.configs import config_instance
inst = config_instance(sys.argv[1] if len(sys.argv) > 1 else "gr17")
genes = torch.rand((30000, 4 * inst.n), dtype=torch.float64, device="cuda")
out = {}
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    D.decode_batch(inst, genes, want_solution=False, out=out)
    torch.cuda.synchronize(); print(f"call {i}: {(time.perf_counter()-t0)*1e3:.2f} ms", flush=True)
