"""Per-launch device timeline of one C3 solve (MP_TIMELINE), for the critical-path analysis in DESIGN §9."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0808_2794_b200 import binding as mp, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED)
A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
x = (torch.rand((1, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
b = (A @ x).t().contiguous().t()
for _ in range(2):
    mp.mp_dsgesv_ex(A, b, None, mp.make_opts(variant=variant))
torch.cuda.synchronize()
os.environ["MP_TIMELINE"] = "gpurun_out/timeline.txt"
_, it, info, rep = mp.mp_dsgesv_ex(A, b, None, mp.make_opts(variant=variant, flags=2))
torch.cuda.synchronize()
print("iters", it, "total", rep.t_total_ms, "factor", rep.t_factor_ms)
