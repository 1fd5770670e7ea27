"""Kernel time per BRKGA generation in a normal (non-ncu) run, from a CUPTI
trace (torch.profiler): python scripts/trace_brkga.py KEY NP GENS"""
import collections
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2602_23685_b200 import brkga as B, configs  # noqa: E402

key, N_p, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = configs.config_instance(key)
B.run_brkga(inst, B.BrkgaParams(population=N_p, generations=2), seed=0)
torch.cuda.synchronize()
walls = {}
for gens in (2, T):
    t = time.perf_counter()
    B.run_brkga(inst, B.BrkgaParams(population=N_p, generations=gens), seed=1)
    torch.cuda.synchronize()
    walls[gens] = time.perf_counter() - t
print(f"{key} N_p={N_p}: {(T - 2) / (walls[T] - walls[2]):.2f} generations/s (wall, no trace)", flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    B.run_brkga(inst, B.BrkgaParams(population=N_p, generations=T), seed=1)
    torch.cuda.synchronize()
tot = collections.defaultdict(lambda: [0, 0.0])
span = [float("inf"), 0.0]
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name][0] += 1
        tot[e.name][1] += e.device_time_total
        span[0] = min(span[0], e.time_range.start)
        span[1] = max(span[1], e.time_range.end)
busy = sum(v[1] for v in tot.values())
print(f"device span {(span[1] - span[0]) / 1e3:.2f} ms, kernel busy {busy / 1e3:.2f} ms over {T} generations")
for name, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{us / 1e3:9.2f} ms  {c:5d}  {us / c:9.1f} us/launch  {name[:90]}")
