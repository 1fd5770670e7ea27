import sys, torch
sys.path.insert(0, ".")
from paper_2602_23685_b200 import configs, device as D
device = torch.device("cuda")
for key in ("eil51", "kroA100"):
    ki = configs.config_instance(key)
    for cnt in (1 << 19, 1 << 20):
        kops = torch.empty((cnt, 2 * ki.n), dtype=torch.int16, device=device)
        klens = torch.empty((cnt, ki.m), dtype=torch.int32, device=device)
        kg = torch.Generator(device=device).manual_seed(int(sys.argv[1]) if len(sys.argv) > 1 else 11)
        for s0 in range(0, cnt, 1 << 16):
            gg = torch.rand((1 << 16, 4 * ki.n), dtype=torch.float64, device=device, generator=kg)
            D.decode_batch(ki, gg, out={"ops": kops[s0:s0 + (1 << 16)], "lens": klens[s0:s0 + (1 << 16)]})
        res = {}
        for _ in range(2):
            D.makespan_batch(ki, kops, klens, mode=0, out=res)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            D.makespan_batch(ki, kops, klens, mode=0, out=res)
        e1.record()
        torch.cuda.synchronize()
        print(key, cnt, 5 * cnt / (e0.elapsed_time(e1) / 1e3) / 1e6, "M/s", (res["status"] != 0).sum().item(), flush=True)
