"""Device-resident C3 solve time (min over reps) and iterations: quick A/B of library variants.
Usage: python tools/probe_c3.py [n] [reps] [label]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0808_2794_b200 import binding as mp, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
label = sys.argv[3] if len(sys.argv) > 3 else ""
g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED)
A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
x = (torch.rand((1, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
b = (A @ x).t().contiguous().t()
X = torch.empty_like(b)
for _ in range(2):
    mp.mp_dsgesv_ex(A, b, X, mp.make_opts(), report=False)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, it, info, _ = mp.mp_dsgesv_ex(A, b, X, mp.make_opts(), report=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
_, it, info, rep = mp.mp_dsgesv_ex(A, b, X, mp.make_opts(flags=4))
torch.cuda.synchronize()
print(f"c3 {label} n={n}: ms={min(ts):.2f} med={sorted(ts)[len(ts) // 2]:.2f} iters={it} info={info} "
      f"factor={rep.t_factor_ms:.2f} refine={rep.t_refine_ms:.2f}", flush=True)
