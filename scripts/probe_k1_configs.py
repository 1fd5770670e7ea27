"""K1 exact-makespan evals/s on every config (decoded random candidates), and
K3 decodes/s -- the small-n side of the north star (shared-memory d)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import configs, device as D  # noqa: E402

for key in (sys.argv[1:] or ("gr17", "eil51", "kroA100", "a280", "dsj1000")):
    inst = configs.config_instance(key)
    N = int(__import__("os").environ.get("NCAND", 1 << 20 if inst.n < 500 else 1 << 19))
    ops = torch.empty((N, 2 * inst.n), dtype=torch.int16, device="cuda")
    lens = torch.empty((N, inst.m), dtype=torch.int32, device="cuda")
    gen = torch.Generator("cuda").manual_seed(5)
    ch = 1 << 16
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dec_ms = 0.0
    D.decode_batch(inst, torch.rand((ch, 4 * inst.n), dtype=torch.float64, device="cuda"),
                   out={"ops": ops[:ch], "lens": lens[:ch]})  # warm: scratch, occupancy plan
    for s in range(0, N, ch):
        g = torch.rand((ch, 4 * inst.n), dtype=torch.float64, device="cuda", generator=gen)
        e0.record()
        D.decode_batch(inst, g, out={"ops": ops[s:s + ch], "lens": lens[s:s + ch]})
        e1.record()
        torch.cuda.synchronize()
        dec_ms += e0.elapsed_time(e1)
    out = {}
    D.makespan_batch(inst, ops, lens, mode=0, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        D.makespan_batch(inst, ops, lens, mode=0, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    bad = int((out["status"] != 0).sum())
    print(f"{key:8s} n={inst.n:4d}: K1 {N / ms / 1e3:8.1f} M evals/s   K3 {N / dec_ms / 1e3:6.2f} M decodes/s  (non-OK statuses: {bad})", flush=True)
