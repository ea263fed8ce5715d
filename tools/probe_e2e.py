"""End-to-end (host A, b, X) solve time at C3 under the current MP_STREAM_* settings, and whether X
matches the device-resident path bitwise.  Usage: python tools/probe_e2e.py [n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0808_2794_b200 import binding as mp, inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED)
dA = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g).t()
x = (torch.rand((1, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
dB = (dA @ x).t().contiguous().t()
Xd, itd, infod, _ = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts())
Xd = Xd.cpu().numpy()
hA = dA.t().contiguous().cpu().pin_memory()
hB = dB.t().contiguous().cpu().pin_memory()
hX = torch.empty((1, n), dtype=torch.float64).pin_memory()
nA, nB, nX = hA.numpy().T, hB.numpy().T, hX.numpy().T
mp.mp_dsgesv_ex(nA, nB, nX, mp.make_opts(), report=False)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, it, info, _ = mp.mp_dsgesv_ex(nA, nB, nX, mp.make_opts())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
gap = float(np.abs(nX - Xd).max() / np.abs(Xd).max())
print(f"e2e n={n} plan={os.environ.get('MP_STREAM_PLAN', '-')} join={os.environ.get('MP_STREAM_JOIN', '-')} "
      f"joined={os.environ.get("MP_STREAM_JOINED", "0")} sm={os.environ.get("MP_H2D_SM", "0")}: ms={min(ts):.2f} (all {[round(t, 2) for t in ts]}) "
      f"iters={it} dev_iters={itd} info={info} x_gap_vs_device={gap:.3g}", flush=True)
if os.environ.get("PROBE_TIMELINE"):
    os.environ["MP_TIMELINE"] = os.environ["PROBE_TIMELINE"]
    _, it, info, rep = mp.mp_dsgesv_ex(nA, nB, nX, mp.make_opts(flags=2))
    torch.cuda.synchronize()
    print("timeline written; total", rep.t_total_ms, flush=True)
