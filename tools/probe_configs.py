"""Run the BASELINE configs C4 (n=49152, nrhs=16) and C5 (n=8192 kappa sweep) once each."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_0808_2794_b200 import binding as mp, inputs
which = sys.argv[1:] or ["c5", "c4"]
if "c5" in which:
    n = 8192
    for kappa in [1e2, 1e4, 1e6, 1e8, 1e10]:
        A, B, X = inputs.conditioned(n, kappa, seed=2794)
        dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
        Xg, it, info, rep = mp.mp_dsgesv_ex(dA, dB)
        torch.cuda.synchronize()
        err = float(np.abs(Xg.cpu().numpy() - X).max() / np.abs(X).max())
        print(json.dumps({"cfg": "C5", "n": n, "kappa": kappa, "iters": it, "info": info, "ms": round(rep.t_total_ms, 2),
                          "fallback_ms": round(rep.t_fallback_ms, 2), "fwd_err": err, "solve_inv": rep.solve_inv}), flush=True)
if "c4" in which:
    n, nrhs = 49152, 16
    g = torch.Generator(device="cuda").manual_seed(2794)
    dA = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()      # column-major view
    Xt = (torch.rand((nrhs, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    dB = (dA @ Xt)
    dB = dB.t().contiguous().t()
    torch.cuda.synchronize()
    for rep_i in range(2):
        Xg, it, info, rep = mp.mp_dsgesv_ex(dA, dB)
        torch.cuda.synchronize()
        print(json.dumps({"cfg": "C4", "n": n, "nrhs": nrhs, "iters": it, "info": info, "ms": round(rep.t_total_ms, 1),
                          "factor_ms": round(rep.t_factor_ms, 1), "refine_ms": round(rep.t_refine_ms, 1),
                          "gflops": round(2 * n**3 / 3 / rep.t_total_ms / 1e6, 1), "solve_inv": rep.solve_inv}), flush=True)
    R = dB - dA @ Xg
    print("C4 max ||r_c|| / (||x_c|| ||A||_F eps sqrt(n)):",
          float((R.norm(dim=0) / (Xg.norm(dim=0) * dA.norm() * 2**-53 * n**0.5)).max()))
