"""e2e scoring of host candidates (schedule.score_host_batch) vs chunk size /
stream count, and the raw pinned H2D bandwidth, at n = 999."""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs, device as D  # noqa: E402

inst = configs.config_instance("dsj1000")
n, m = inst.n, inst.m
N = 1 << 18
g = torch.rand((1 << 16, 4 * n), dtype=torch.float64, device="cuda")
ops = torch.empty((N, 2 * n), dtype=torch.int16, device="cuda")
lens = torch.empty((N, m), dtype=torch.int32, device="cuda")
for s in range(0, N, 1 << 16):
    D.decode_batch(inst, g, out={"ops": ops[s:s + (1 << 16)], "lens": lens[s:s + (1 << 16)]})
h_ops = torch.empty(ops.shape, dtype=torch.int16, pin_memory=True)
h_lens = torch.empty(lens.shape, dtype=torch.int32, pin_memory=True)
h_ops.copy_(ops)
h_lens.copy_(lens)
torch.cuda.synchronize()
# raw H2D
buf = torch.empty_like(ops)
for _ in range(2):
    buf.copy_(h_ops, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    buf.copy_(h_ops, non_blocking=True)
torch.cuda.synchronize()
print(f"raw pinned H2D: {5 * h_ops.numel() * 2 / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
for chunk in (1 << 14, 1 << 15, 1 << 16, 1 << 17):
    for nst in (2, 3, 4):
        D_N = D.__dict__
        D.N_STREAMS = nst
        D.score_host_batch(inst, h_ops, h_lens, chunk=chunk)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(4):
            D.score_host_batch(inst, h_ops, h_lens, chunk=chunk)
        dt = (time.perf_counter() - t) / 4
        print(f"chunk {chunk:6d} streams {nst}: {N / dt / 1e6:6.2f} M evals/s  ({N * 2 * n * 2 / dt / 1e9:5.1f} GB/s ops)",
              flush=True)
