"""K2 (two_pass_estimate) evals/s on decoded dsj1000 candidates + one cross-LS pass."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import alns as A, configs, device as D, localsearch as LS  # noqa: E402
inst = configs.config_instance("dsj1000")
N = 1 << 18
g = torch.rand((N, 4 * inst.n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
dec = D.decode_batch(inst, g, op_dtype=torch.int16)
del g
out = {}
D.makespan_batch(inst, dec["ops"], dec["lens"], mode=2, out=out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    D.makespan_batch(inst, dec["ops"], dec["lens"], mode=2, out=out)
e1.record()
torch.cuda.synchronize()
print(f"K2 two-pass: {3 * N / e0.elapsed_time(e1) / 1e3:.1f} M evals/s", flush=True)
sol = A.construct_initial(inst)
o, l = sol.to_arrays(inst.n)
t = time.perf_counter()
LS.cross_agent_relocation_batch(inst, o[None, :2 * inst.n], l[None])
torch.cuda.synchronize()
print(f"cross LS pass at n=999: {time.perf_counter() - t:.2f}s", flush=True)
