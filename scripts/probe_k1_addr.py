"""Diagnostic: is the small-n K1 rate data- or placement-dependent?"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs, device as D  # noqa: E402

inst = configs.config_instance("eil51")
N, ch = 1 << 20, 1 << 16
ops = torch.empty((N, 2 * inst.n), dtype=torch.int16, device="cuda")
lens = torch.empty((N, inst.m), dtype=torch.int32, device="cuda")
gen = torch.Generator("cuda").manual_seed(5)
for s in range(0, N, ch):
    g = torch.rand((ch, 4 * inst.n), dtype=torch.float64, device="cuda", generator=gen)
    D.decode_batch(inst, g, out={"ops": ops[s:s + ch], "lens": lens[s:s + ch]})
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def rate(o, l, label):
    out = {}
    D.makespan_batch(inst, o, l, mode=0, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        D.makespan_batch(inst, o, l, mode=0, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label:24s} {o.shape[0] * 5 / e0.elapsed_time(e1) / 1e3:7.1f} M evals/s", flush=True)


rate(ops, lens, "full 2^20")
rate(ops[:N // 2], lens[:N // 2], "first half")
rate(ops[N // 2:], lens[N // 2:], "second half")
c_ops, c_lens = ops.clone(), lens.clone()
rate(c_ops, c_lens, "clone full")
rate(c_ops[:N // 2].clone(), c_lens[:N // 2].clone(), "clone first half")
rate(ops, lens, "full again")
