"""mp_dsgesv time at n=16384 for several panel widths (opts.nb)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0808_2794_b200 import binding as mp, inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A, B, _ = inputs.gaussian(n, nrhs=1, seed=2794)
dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
for nb in [int(x) for x in (sys.argv[2:] or ["192", "256", "320", "384", "512"])]:
    best = None
    for rep in range(3):
        X, it, info, r = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(nb=nb))
        torch.cuda.synchronize()
        best = r if best is None or r.t_total_ms < best.t_total_ms else best
    print(json.dumps({"nb": nb, "iters": it, "total_ms": round(best.t_total_ms, 2), "factor_ms": round(best.t_factor_ms, 2),
                      "refine_ms": round(best.t_refine_ms, 2)}), flush=True)
