"""Refinement time vs nrhs (n = 16384 default): exercises the R = 1 / 4 / 16 sweep instantiations."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0808_2794_b200 import binding as mp, inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for nrhs in (1, 4, 8, 16):
    A, B, _ = inputs.gaussian(n, nrhs=nrhs, seed=2794)
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    for rep in range(2):
        X, it, info, r = mp.mp_dsgesv_ex(dA, dB)
    torch.cuda.synchronize()
    print(json.dumps({"n": n, "nrhs": nrhs, "iters": it, "info": info, "total_ms": round(r.t_total_ms, 2),
                      "factor_ms": round(r.t_factor_ms, 2), "refine_ms": round(r.t_refine_ms, 2)}), flush=True)
