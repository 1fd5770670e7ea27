"""A few BRKGA generations at paper scale for the launch list:
python scripts/profile_brkga.py KEY NP GENS"""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import brkga as B, configs  # noqa: E402
key, N_p, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = configs.config_instance(key)
B.run_brkga(inst, B.BrkgaParams(population=N_p, generations=1), seed=0)
torch.cuda.synchronize()
t = time.perf_counter()
B.run_brkga(inst, B.BrkgaParams(population=N_p, generations=T), seed=1)
torch.cuda.synchronize()
print(f"{key} N_p={N_p}: {T / (time.perf_counter() - t):.2f} generations/s", flush=True)
