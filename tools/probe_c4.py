"""C4 (n = 49152, nrhs = 16) on one GPU: time, the trailing update's achieved rate inside the solve
(flags bits 1|3: events around the trailing-update and residual launches only) and, with `timeline`,
a fully instrumented per-launch device timeline (MP_TIMELINE) for the per-step critical-path analysis.
Usage: python tools/probe_c4.py [n] [nrhs] [timeline]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0808_2794_b200 import binding as mp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
timeline = len(sys.argv) > 3 and sys.argv[3] == "timeline"
NB = int(os.environ.get("PROBE_NB", "0"))
NAMES = ["demote", "panel", "laswp", "trsm", "gemm", "solve", "residual", "trail"]
g = torch.Generator(device="cuda").manual_seed(2794)
dA = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
Xt = (torch.rand((nrhs, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
dB = (dA @ Xt).t().contiguous().t()
torch.cuda.synchronize()
for i in range(2):
    Xg, it, info, rep = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(flags=2 | 8, nb=NB))
    torch.cuda.synchronize()
    k = {NAMES[c]: [round(rep.k_ms[c], 2), int(rep.k_launches[c]), round(rep.k_work[c] / max(rep.k_ms[c], 1e-9) / 1e9, 1)]
         for c in range(8) if rep.k_launches[c]}
    print(json.dumps({"cfg": "C4", "n": n, "nrhs": nrhs, "nb": rep.nb, "iters": it, "info": info, "ms": round(rep.t_total_ms, 1),
                      "factor_ms": round(rep.t_factor_ms, 1), "refine_ms": round(rep.t_refine_ms, 1),
                      "gflops": round(2 * n ** 3 / 3 / rep.t_total_ms / 1e6, 1),
                      "classes [ms, launches, Gwork/s]": k}), flush=True)
if timeline:
    os.environ["MP_TIMELINE"] = "gpurun_out/timeline_c4.txt"
    Xg, it, info, rep = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(flags=2))
    torch.cuda.synchronize()
    print("instrumented: total", round(rep.t_total_ms, 1), "factor", round(rep.t_factor_ms, 1))
