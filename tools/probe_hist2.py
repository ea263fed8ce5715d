"""Residual-ratio histories at n (default 16384) for several MP_TF32_TERMS4_FRAC settings and seeds."""
import os, sys, subprocess, json
code = r'''
import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_0808_2794_b200 import binding as mp, inputs
n = int(sys.argv[1]); seed = int(sys.argv[2])
A, B, _ = inputs.gaussian(n, nrhs=1, seed=seed)
dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
X, it, info, r = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts())
torch.cuda.synchronize()
print(it, [f"{v:.3g}" for v in r.history()], round(r.t_total_ms, 2))
'''
n = sys.argv[1] if len(sys.argv) > 1 else "16384"
for f in ["0", "0.3", "0.5", "1.0"]:
    for seed in ["2794", "1", "2"]:
        env = dict(os.environ, MP_TF32_TERMS4_FRAC=f)
        out = subprocess.run([sys.executable, "-c", code, n, seed], env=env, capture_output=True, text=True).stdout.strip()
        print("frac", f, "seed", seed, out, flush=True)
