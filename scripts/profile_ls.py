"""One cross-LS pass at dsj1000 for ncu (vrp_ls_build + K2 chunks)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2602_23685_b200 import alns as A, configs, localsearch as LS  # noqa: E402
inst = configs.config_instance("dsj1000")
sol = A.construct_initial(inst)
o, l = sol.to_arrays(inst.n)
LS.cross_agent_relocation_batch(inst, o[None, :2 * inst.n], l[None])
torch.cuda.synchronize()
