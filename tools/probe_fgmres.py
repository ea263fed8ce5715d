"""One FGMRES(10)-GMRES_SP(20) solve at n = 16384 on the GPU (for ncu captures of the G7 kernel)."""
import math
import sys

import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0808_2794_b200 import binding as mp, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED + 11)
A = (torch.randn((n, n), dtype=torch.float64, device=dev, generator=g) / math.sqrt(n)).t()
A.diagonal().add_(2.5)
x = (torch.rand((1, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
b = (A @ x).t().contiguous().t()
for _ in range(2):
    _, it, info, rep = mp.mp_fgmres_ex(A, b, m_out=10, m_in=20)
torch.cuda.synchronize()
_, it, info, rep = mp.mp_fgmres_ex(A, b, m_out=10, m_in=20, opts=mp.make_opts(flags=2))
torch.cuda.synchronize()
k = rep.kernels()
sv = k["solve"]
print("iters", it, "info", info, "ms", round(rep.t_total_ms, 3), "inner ms/cycle", round(sv["ms"] / sv["launches"], 4),
      "GB/s", round(sv["work"] / sv["ms"] / 1e6, 1))
