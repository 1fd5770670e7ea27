"""K1 time per 65,536-candidate chunk of a decoded eil51 set (diagnostic)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs, device as D  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "eil51"
inst = configs.config_instance(key)
N, ch = 1 << 19, 1 << 16
ops = torch.empty((N, 2 * inst.n), dtype=torch.int16, device="cuda")
lens = torch.empty((N, inst.m), dtype=torch.int32, device="cuda")
gen = torch.Generator("cuda").manual_seed(5)
for s in range(0, N, ch):
    g = torch.rand((ch, 4 * inst.n), dtype=torch.float64, device="cuda", generator=gen)
    D.decode_batch(inst, g, out={"ops": ops[s:s + ch], "lens": lens[s:s + ch]})
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    for s in range(0, N, ch):
        out = {}
        D.makespan_batch(inst, ops[s:s + ch], lens[s:s + ch], mode=0, out=out)
        torch.cuda.synchronize()
        e0.record()
        D.makespan_batch(inst, ops[s:s + ch], lens[s:s + ch], mode=0, out=out)
        e1.record()
        torch.cuda.synchronize()
        print(rep, s // ch, f"{e0.elapsed_time(e1):.3f} ms", flush=True)
for sz in (1 << 18, 1 << 19):
    out = {}
    D.makespan_batch(inst, ops[:sz], lens[:sz], mode=0, out=out)
    torch.cuda.synchronize()
    e0.record()
    D.makespan_batch(inst, ops[:sz], lens[:sz], mode=0, out=out)
    e1.record()
    torch.cuda.synchronize()
    print("prefix", sz, f"{e0.elapsed_time(e1):.3f} ms", flush=True)
