import os, sys, json
sys.path.insert(0, '/root/repo')
import torch
from paper_0808_2794_b200 import binding as mp, inputs
A, B, _ = inputs.gaussian(16384, nrhs=1, seed=2794)
dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
for fl, name in [(0, "inv"), (32, "subst")]:
    X, it, info, r = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(flags=fl))
    torch.cuda.synchronize()
    print(name, it, [f"{v:.3g}" for v in r.history()], r.solve_inv)
X, it, info, r = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(variant=mp.MP_VARIANT_FFMA))
torch.cuda.synchronize()
print("ffma", it, [f"{v:.3g}" for v in r.history()])
