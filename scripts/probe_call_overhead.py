import sys, time, torch
sys.path.insert(0, ".")
from paper_2602_23685_b200 import configs, device as D
ki = configs.config_instance("eil51")
ops = torch.zeros((1024, 100), dtype=torch.int16, device="cuda")
lens = torch.zeros((1024, ki.m), dtype=torch.int32, device="cuda")
res = {}
D.makespan_batch(ki, ops, lens, mode=0, out=res); torch.cuda.synchronize()
for label in ("makespan_batch",):
    t = time.perf_counter()
    for _ in range(200):
        D.makespan_batch(ki, ops, lens, mode=0, out=res)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(label, "cpu per call us", (t1 - t) / 200 * 1e6, "incl sync", (time.perf_counter() - t) / 200 * 1e6)
import cProfile, pstats
cProfile.run("for _ in range(200): D.makespan_batch(ki, ops, lens, mode=0, out=res)", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumtime").print_stats(12)
