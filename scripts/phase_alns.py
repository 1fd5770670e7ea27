"""Per-phase clocks of the ALNS kernel (needs a -DVRP_PHASE_TIMERS build via VRP_LIB):
python scripts/phase_alns.py KEY W ITERS"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import alns as A, configs  # noqa: E402
key, W, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = configs.config_instance(key)
init = A.construct_initial(inst)
prm = A.AlnsParams(max_iter=max(iters, 8), pickup_reposition_interval=10**9, cross_agent_interval=10**9)
ws = [A._Worker(inst, prm, A.worker_seed(1, i), init, None, None, i) for i in range(W)]
dw = A._DeviceWorkers(inst, prm, ws)
dw._buffers(max(iters, 8))
dw.DV.alns_iterate(inst, dw.cparams, dw.g_rec, dw.g_cur_ops, dw.g_cur_lens, dw.g_best_ops, dw.g_best_lens,
                   dw.g_q, 1, iters, dw.t_it, dw.t_z, dw.r_it, dw.r_val)
torch.cuda.synchronize()
t = dw.t_z[:, :6].cpu().numpy()
tot = t[:, :4].sum(1)
names = ["destroy+remove", "rebuild+compact", "reinsert_core", "replay"]
print(f"{key} W={W} iters={iters}: mean clocks/iter {tot.mean() / iters:.3e}")
for j, nm in enumerate(names):
    print(f"  {nm:16s} {100 * t[:, j].sum() / tot.sum():5.1f}%")
print(f"  removed per iteration {t[:, 4].mean() / iters:.1f}, customer_options calls ~ {t[:, 5].mean() / iters:.0f}")
