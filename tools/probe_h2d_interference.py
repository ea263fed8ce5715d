"""Does a concurrent H2D copy (PCIe DMA into HBM) slow the device-resident factorisation?  C3 solve
time alone and with a copy stream running (checked to still be running when the solve ends), plus
per-class kernel averages from an instrumented solve in both conditions.
Usage: python tools/probe_h2d_interference.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0808_2794_b200 import binding as mp, inputs

n = 16384
g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED)
A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
x = (torch.rand((1, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
b = (A @ x).t().contiguous().t()
X = torch.empty_like(b)
host = torch.empty((2048, n), dtype=torch.float64).pin_memory()      # 256 MB
dst = torch.empty((2048, n), dtype=torch.float64, device="cuda")
cs = torch.cuda.Stream()
ms_ = torch.cuda.Stream()
NAMES = ["demote", "panel", "laswp", "trsm", "gemm", "solve", "residual", "trail"]


def run(bg, flags):
    torch.cuda.synchronize()
    if bg:
        with torch.cuda.stream(cs):
            for _ in range(24):                      # ~6 GB: longer than the solve
                dst.copy_(host, non_blocking=True)
    with torch.cuda.stream(ms_):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, it, info, rep = mp.mp_dsgesv_ex(A, b, X, mp.make_opts(flags=flags), report=flags != 0)
        e1.record()
    e1.synchronize()
    busy = bg and not cs.query()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), it, busy, rep


for _ in range(2):
    run(False, 0)
for bg in (False, True, False, True):
    t, it, busy, _ = run(bg, 0)
    print(f"background copy={bg} (still running at solve end: {busy}): solve {t:.2f} ms iters {it}", flush=True)
for bg in (False, True):
    t, it, busy, rep = run(bg, 2)
    avg = {NAMES[c]: round(1e3 * rep.k_ms[c] / max(1, rep.k_launches[c]), 1) for c in range(8) if rep.k_launches[c]}
    print(f"instrumented, background copy={bg} (running at end: {busy}): {t:.2f} ms, avg us per launch {avg}", flush=True)
