"""Per-kernel-class timing of one mp_dsgesv solve at several n (CUDA events around every launch)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_0808_2794_b200 import binding as mp, inputs
variant = mp.MP_VARIANT_3XTF32 if "--ffma" not in sys.argv else mp.MP_VARIANT_FFMA
ns = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1024, 4096, 8192, 16384]
flags = 0 if "--noprof" in sys.argv else 2
for n in ns:
    A, B, _ = inputs.gaussian(n, nrhs=1, seed=2794)
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    for rep in range(2):
        X, it, info, r = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(variant=variant, flags=flags))
    torch.cuda.synchronize()
    k = r.kernels()
    row = {c: (round(v["ms"], 3), v["launches"], round(1e3 * v["ms"] / max(1, v["launches"]), 1)) for c, v in k.items()}
    print(json.dumps({"n": n, "iters": it, "total_ms": round(r.t_total_ms, 3), "factor_ms": round(r.t_factor_ms, 3),
                      "refine_ms": round(r.t_refine_ms, 3), "classes(ms,launches,us/launch)": row}), flush=True)
