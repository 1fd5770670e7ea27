import sys, time
sys.path.insert(0, ".")
import torch
from paper_2602_23685_b200 import alns as A, configs
inst = configs.config_instance("kroA100")
init = A.construct_initial(inst)
for max_iter, ls in ((200, False), (200_000, False), (200_000, True)):
    kw = {} if ls else {"pickup_reposition_interval": 10**9, "cross_agent_interval": 10**9}
    prm = A.AlnsParams(max_iter=max_iter, **kw)
    ws = [A._Worker(inst, prm, A.worker_seed(0, i), init, None, None, i) for i in range(296)]
    dw = A._DeviceWorkers(inst, prm, ws)
    t0 = time.perf_counter()
    log = []
    def stop():
        zs = sorted(w.z_best for w in ws)
        log.append((dw.iterations, round(time.perf_counter() - t0, 1), zs[0], zs[len(zs)//2], ws[0].z, ws[0].temperature))
        return dw.iterations >= 200
    dw.drive(stop=stop, max_stretch=25)
    print(max_iter, ls, log, flush=True)
