"""Diagnostic: K1 rate vs where the op buffer lands in device memory
(fresh allocation vs after torch.cuda.empty_cache()).
python scripts/probe_k1_bench_ctx.py"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
sys.argv = [sys.argv[0]]
sys.path.insert(0, "scripts")
from probe_k1_order import k1  # noqa: E402

for key, cnt in (("eil51", 1 << 20), ("dsj1000", 1 << 19)):
    k1(key, cnt, f"{key} fresh")
    k1(key, cnt, f"{key} reuse")
    torch.cuda.empty_cache()
    k1(key, cnt, f"{key} after empty_cache")
    torch.cuda.empty_cache()
    k1(key, cnt, f"{key} after empty_cache 2")
