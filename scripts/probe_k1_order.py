import sys
sys.path.insert(0, ".")
import torch
from paper_2602_23685_b200 import configs, device as D

def k1(key, cnt, label):
    ki = configs.config_instance(key)
    kops = torch.empty((cnt, 2 * ki.n), dtype=torch.int16, device="cuda")
    klens = torch.empty((cnt, ki.m), dtype=torch.int32, device="cuda")
    kg = torch.Generator(device="cuda").manual_seed(11)
    for s0 in range(0, cnt, 1 << 16):
        gg = torch.rand((1 << 16, 4 * ki.n), dtype=torch.float64, device="cuda", generator=kg)
        D.decode_batch(ki, gg, out={"ops": kops[s0:s0 + (1 << 16)], "lens": klens[s0:s0 + (1 << 16)]})
    res = {}
    for _ in range(2):
        D.makespan_batch(ki, kops, klens, mode=0, out=res)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5):
        D.makespan_batch(ki, kops, klens, mode=0, out=res)
    e1.record(); torch.cuda.synchronize()
    print(f"{label:30s} {5 * cnt / (e0.elapsed_time(e1) / 1e3) / 1e6:8.1f} M evals/s", flush=True)

order = sys.argv[1] if len(sys.argv) > 1 else ""
if order == "dsj_first":
    k1("dsj1000", 1 << 18, "dsj1000 2^18")
k1("eil51", 1 << 20, "eil51 2^20")
k1("kroA100", 1 << 20, "kroA100 2^20")
k1("eil51", 1 << 20, "eil51 2^20 again")
if order == "alns_first":
    from paper_2602_23685_b200 import alns as A
    inst = configs.config_instance("eil51")
    init = A.construct_initial(inst)
    prm = A.AlnsParams(max_iter=100, pickup_reposition_interval=10**9, cross_agent_interval=10**9)
    ws = [A._Worker(inst, prm, A.worker_seed(3, i), init, None, None, i) for i in range(1184)]
    dw = A._DeviceWorkers(inst, prm, ws)
    dw.run(1, 5)
    torch.cuda.synchronize()
    k1("eil51", 1 << 20, "eil51 2^20 after ALNS")
    del dw, ws
    torch.cuda.synchronize()
    k1("eil51", 1 << 20, "eil51 2^20 after del")
if order == "repair_first":
    import numpy as np
    sys.path.insert(0, "tests")
    sys.path.insert(0, "tests/golden")
    from oracle import oracle as O
    import inputs as I
    from paper_2602_23685_b200 import insertion as INS
    inst = configs.config_instance("eil51")
    cnt = 1024
    genes = I.chromosomes(inst.n, cnt, (7, 7))
    dec = O.decode_batch(inst, genes)
    k1("eil51", 1 << 20, "eil51 after O.decode")
    parts, plens, rem = [], [], []
    for i in range(cnt):
        pick = I.philox(8, i).choice(np.arange(1, inst.n + 1), size=5, replace=False)
        o, l, r = O.remove_customers(inst, dec["ops"][i], dec["lens"][i], pick)
        parts.append(o[:2 * inst.n]); plens.append(l); rem.append(r)
    parts, plens = np.stack(parts), np.stack(plens)
    rks = [(0, 2, 3, inst.m)[i % 4] for i in range(cnt)]
    INS.reinsert_batch(inst, parts, plens, rem, rks, [I.philox(9, i) for i in range(cnt)])
    torch.cuda.synchronize()
    k1("eil51", 1 << 20, "eil51 after reinsert")
