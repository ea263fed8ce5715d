"""FP64 path probe: mp_dgesv per-kernel-class breakdown (flags bit 1) at n, and cuSOLVER
dgetrf+dgetrs (torch.linalg.lu_factor / lu_solve, context only — never on the product path)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_0808_2794_b200 import binding as mp, inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A, B, X = inputs.gaussian(n, nrhs=1, seed=2794)
dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
out = {"n": n}
for name, flags in (("plain", 0), ("profiled", 2)):
    Xd, info, rep = mp.mp_dgesv_ex(dA, dB, opts=mp.make_opts(flags=flags))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Xd, info, rep = mp.mp_dgesv_ex(dA, dB, opts=mp.make_opts(flags=flags))
    e1.record()
    torch.cuda.synchronize()
    out[name] = {"ms": e0.elapsed_time(e1), "t_factor_ms": rep.t_factor_ms, "info": info}
    if flags:
        out[name]["kernels"] = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                                    "tflops_or_gbs": round(v["work"] / v["ms"] / 1e9, 2) if v["ms"] else None}
                                for k, v in rep.kernels().items()}
# cuSOLVER context (torch.linalg -> cusolverDnXgetrf / getrs), fp64
At = dA.contiguous()
for _ in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    LU, piv = torch.linalg.lu_factor(At)
    Xc = torch.linalg.lu_solve(LU, piv, dB.contiguous())
    e1.record()
    torch.cuda.synchronize()
out["cusolver_dgetrf_dgetrs_ms"] = e0.elapsed_time(e1)
out["cusolver_tflops"] = 2 * n ** 3 / 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps(out, indent=1))

# the binary64 trailing update alone: M = N = n - 256, K = 256, full GPU
W = torch.randn(n, n, dtype=torch.float64, device="cuda")
for pipe, name in ((1, "dmma"), (2, "dfma")):
    M = N = n - 256
    mp.mp_kernel_schur_update_f64(W, 256, 256, 0, M, N, 256, pipe)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        mp.mp_kernel_schur_update_f64(W, 256, 256, 0, M, N, 256, pipe)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out["gemm_" + name] = {"ms": ms, "tflops": 2.0 * M * N * 256 / (ms * 1e-3) / 1e12}
print(json.dumps({k: out[k] for k in out if k.startswith("gemm")}))
