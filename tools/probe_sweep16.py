"""One mp_dsgesv at n = 16384 with 16 right-hand sides (ncu capture of the R = 16 sweeps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0808_2794_b200 import binding as mp, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED)
A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
X = (torch.rand((nrhs, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
B = (A @ X).t().contiguous().t()
_, it, info, rep = mp.mp_dsgesv_ex(A, B, None, mp.make_opts(flags=16))
torch.cuda.synchronize()
print("iters", it, "info", info, "refine", rep.t_refine_ms)
