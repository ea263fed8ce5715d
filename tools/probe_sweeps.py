"""Triangular-sweep cost against the number of right-hand sides (C3 / C4 sizes): ms per sweep pair."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0808_2794_b200 import binding as mp, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED)
A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
for nrhs in [1, 2, 4, 8, 9, 16]:
    X = (torch.rand((nrhs, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (A @ X).t().contiguous().t()
    mp.mp_dsgesv_ex(A, B, None, mp.make_opts())
    torch.cuda.synchronize()
    _, it, info, rep = mp.mp_dsgesv_ex(A, B, None, mp.make_opts(flags=2))
    torch.cuda.synchronize()
    k = rep.kernels()
    sv, rs = k["solve"], k["residual"]
    pairs = sv["launches"] - 1        # the inverses launch is a 'solve' record too
    print(f"n={n} nrhs={nrhs} iters={it} total={rep.t_total_ms:.1f} refine={rep.t_refine_ms:.2f} "
          f"solve_ms={sv['ms']:.2f} launches={sv['launches']} per_pair={sv['ms'] / max(1, pairs):.3f} "
          f"residual_ms={rs['ms']:.2f}", flush=True)
