#!/usr/bin/env python
"""bench.py — FP64-accurate mixed-precision solve throughput on B200 (BASELINE.json metric).

One "step" = one full mp_dsgesv solve (Alg. 1 of arXiv 0808.2794: demote, binary32
blocked GEPP, x0, binary64 residual / binary32 correction loop until B:5's test)
of the C3 workload: n = 16384, A i.i.d. N(0,1) fp64 (2.1 GB > L2), x_true U[-1,1],
b = A x_true, nrhs = 1.  Inputs are resident in HBM when the timed region starts;
A (2.1 GB) is larger than L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]

value        = 2 n^3 / 3 flops per solve x solves (all ranks) / device time (max over ranks), GFLOP/s
e2e          = same metric through the C-ABI with HOST buffers (H2D of A, b and D2H of x inside)
speedup_vs_fp64 = t(mp_dgesv) / t(mp_dsgesv) on the same inputs (B:5; the paper's T3 analog)
roofline     = dominant kernel class (CUDA events around each launch inside the timed region)
cpu_baseline = the CPU oracle (oracle/oracle.c) on a bounded sample, rank 0, N = 1 only
--impl reference: this tier's reference arm is the oracle itself (no reference package exists).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_0808_2794_b200 import inputs  # noqa: E402

WORKLOAD = "C3: n=16384 dense nonsymmetric, A iid N(0,1) fp64, x_true U[-1,1], b=A x_true, nrhs=1"
METRIC = "FP64-accurate solve GFLOP/s (2n^3/3 per solve), mixed fp32 LU + fp64 refinement"


def flops(n: int) -> float:
    return 2.0 * n ** 3 / 3.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms around the timed region.

    nvidia-smi needs a few hundred ms to start, longer than a short timed region, so the sampler
    is started before the warm-up (start()); the summary uses the samples stamped inside the timed
    window [begin, end] widened by 150 ms on each side, and waits (up to 2 s) for one sample after
    the window so that a short region is never unsampled."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.t_begin = self.t_end = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append((time.perf_counter(), parts))

    # timed window
    def __enter__(self):
        if self.proc is None:
            self.start()
        self.t_begin = time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.t_end = time.perf_counter()
        deadline = self.t_end + 2.0
        while self.proc and time.perf_counter() < deadline and not any(t > self.t_end for t, _ in self.rows):
            time.sleep(0.02)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        lo = (self.t_begin or 0.0) - 0.15
        hi = (self.t_end or 1e30) + 0.15
        rows = [r for t, r in self.rows if lo <= t <= hi]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- reference arm (the oracle)
def cpu_oracle_sample(n_cpu: int, seed: int):
    import oracle
    oracle.build()
    A, B, _ = inputs.gaussian(n_cpu, nrhs=1, seed=seed)
    t0 = time.perf_counter()
    r = oracle.dsgesv(A, B)
    dt = time.perf_counter() - t0
    return dt, r, oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    n_cpu = args.cpu_n
    times = []
    for i in range(args.warmup + args.steps):
        dt, r, threads = cpu_oracle_sample(n_cpu, inputs.BASE_SEED)
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    v = flops(n_cpu) / t / 1e9
    out = {"metric": METRIC, "value": round(v, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32+f64 (CPU oracle: plain binary32 GEPP)", "data": "synthetic", "impl": "reference",
           "config": {"workload": WORKLOAD, "n": args.n, "nrhs": 1, "sample_n": n_cpu},
           "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                            "sample": f"one full oracle_dsgesv solve per step at n={n_cpu} (same generator), "
                                      f"iters={r.iters}"},
           "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm, N GPUs
def run_distributed(args, rank, world, dev, dist, mp, variant):
    """C3 strong scaling (B:9): ONE n x n system distributed 1D block-cyclic by column blocks of nb
    over the N ranks; panel broadcasts / residual all-reduces over NCCL."""
    import torch
    from paper_0808_2794_b200 import dist as pd
    n, nrhs = args.n, args.nrhs
    nb = args.nb if args.nb > 0 else 256
    uid = pd.exchange_uid(rank, mp.mp_get_unique_id)
    comm = mp.mp_comm_init(world, rank, uid)
    cols = mp.local_columns(n, nb, world, rank)
    Al = pd.gen_local_A(n, nb, world, rank, inputs.BASE_SEED, device=str(dev))
    Xt = pd.gen_xtrue(n, nrhs, inputs.BASE_SEED, device=str(dev))
    B = pd.distributed_rhs(Al, Xt, cols).t().contiguous().t()
    X = torch.empty((nrhs, n), dtype=torch.float64, device=dev).t()
    torch.cuda.synchronize()
    opts = mp.make_opts(nb=nb, variant=variant, flags=2 | 4 | 8)

    def barrier():
        if dist is not None:
            dist.barrier()

    def solve(o=opts, report=True):
        return mp.mp_dsgesv_1dbc_ex(comm, n, nb, Al, B, X, o, report)

    clk = ClockSampler(dev.index).start()                         # running before the warm-up
    for _ in range(args.warmup):
        _, it, info, _ = solve()
    assert info == 0 and it >= 0, (it, info)
    mp.mp_profile_collect()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    barrier()
    torch.cuda.synchronize()
    with clk:
        e0.record(stream)
        for _ in range(args.steps):
            _, it, info, rep = solve()
            reps.append((it, info, rep))
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()

    def maxr(v):
        if dist is None:
            return v
        t = torch.tensor([v], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_step = maxr(e0.elapsed_time(e1)) / args.steps
    value = flops(n) / (ms_step / 1e3) / 1e9                  # one solve per step for the whole job
    kern = mp.mp_profile_collect().kernels()
    pk, pk_src = peaks()
    tf32_peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1400.0)) * (1.1 / 2.25)
    roof = None
    if "trail" in kern and kern["trail"]["ms"] > 0:
        d = kern["trail"]
        mult = 3.0 if args.variant == "3xtf32" else 1.0
        ach = mult * d["work"] / (d["ms"] / 1e3) / 1e12
        peak = tf32_peak if args.variant == "3xtf32" else 148 * 128 * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        roof = {"kernel": "trailing Schur update (K5, %s), rank %d" % (args.variant, rank),
                "bound": "tensor" if mult == 3.0 else "alu", "achieved": round(ach, 2), "peak": round(peak, 1),
                "unit": "TFLOP/s", "frac": round(ach / peak, 4), "traffic": None, "peak_source": pk_src}
    # binary64 distributed path (speedup denominator)
    fp64_ms = None
    if args.fp64_steps > 0:
        mp.mp_dgesv_1dbc(comm, n, nb, Al, B, X)
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.fp64_steps):
            mp.mp_dgesv_1dbc(comm, n, nb, Al, B, X)
        f1.record(stream)
        torch.cuda.synchronize()
        fp64_ms = maxr(f0.elapsed_time(f1)) / args.fp64_steps
    # end to end: pinned host A_local / B in, X out, copies inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        hA = Al.t().contiguous().cpu().pin_memory()
        hB = B.t().contiguous().cpu().pin_memory()
        hX = torch.empty((nrhs, n), dtype=torch.float64).pin_memory()
        dA2 = torch.empty_like(Al.t().contiguous())
        dB2 = torch.empty_like(B.t().contiguous())
        barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.e2e_steps):
            dA2.copy_(hA, non_blocking=True)
            dB2.copy_(hB, non_blocking=True)
            Xo, _, _, _ = mp.mp_dsgesv_1dbc_ex(comm, n, nb, dA2.t(), dB2.t(), X, mp.make_opts(nb=nb, variant=variant),
                                                False)
            hX.copy_(Xo.t(), non_blocking=True)
        g1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = maxr(g0.elapsed_time(g1)) / args.e2e_steps
        e2e = {"value": round(flops(n) / (e2e_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 8 * n * n + 8 * n * nrhs * world, "d2h_bytes_per_step": 8 * n * nrhs * world,
               "ms_per_step": round(e2e_ms, 3)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        dt, r, threads = cpu_oracle_sample(args.cpu_n, inputs.BASE_SEED)
        cpu = {"value": round(flops(args.cpu_n) / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
               "kind": "oracle", "sample": f"one full oracle_dsgesv solve at n={args.cpu_n} (same generator family, "
                                           f"{dt:.1f} s, iters={r.iters})"}
    if rank == 0:
        iters = [r[0] for r in reps]
        out = {"metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": dtype_label(args.variant),
               "data": "synthetic (per-block seeded N(0,1) columns, x_true U[-1,1], b = A x_true)",
               "config": {"workload": WORKLOAD, "n": n, "nrhs": nrhs, "nb": nb, "variant": args.variant,
                          "iters": iters, "l2": "inputs larger than L2",
                          "parallelism": f"1D block-cyclic column blocks of {nb} over {world} GPU(s), NCCL"},
               "speedup_vs_fp64": round(fp64_ms / ms_step, 3) if fp64_ms else None,
               "fp64_ms_per_step": round(fp64_ms, 3) if fp64_ms else None,
               "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
               "gpu_launches": sum(r[2].kernel_launches for r in reps)}
        print(json.dumps(out), flush=True)
    mp.mp_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- our arm
def _gemm_traffic():
    """dram bytes (read + write) of one trailing-update launch from the committed ncu --set full
    capture of the current code (profiles/r02_gemm_full_pair.json), with its algorithmic bytes; None if absent."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_gemm_full_pair.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    return {"bytes": d["dram_read_bytes"] + d["dram_write_bytes"], "algorithmic_bytes": d["algorithmic_bytes"],
            "ratio": d["traffic_over_algorithmic"], "launch": "M=N=%d K=%d (%s)" % (d["M"], d["K"], os.path.basename(p))}


def _gemm_alone(peak: float):
    """The same kernel with the whole GPU (one trailing-update launch outside the look-ahead), from the
    committed ncu capture (profiles/r02_gemm_full_pair.json; ncu's own duration, so context, not the bench value)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_gemm_full_pair.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    return {"achieved": d["achieved_tflops_3x"], "frac": round(d["achieved_tflops_3x"] / peak, 4), "sms": d["grid"],
            "tc_pipe_active_pct": d.get("sm__pipe_tc_cycles_active_pct"),
            "launch": "M=N=%d K=%d, %.0f us (%s)" % (d["M"], d["K"], d["duration_us"], os.path.basename(p))}


def dtype_label(variant: str) -> str:
    """The arithmetic the path computes in: binary32 LU (its O(n^3) update on 3xTF32 tcgen05 tensor
    cores, or FP32 FFMA), binary64 residual / update / test."""
    return "f32 LU (3xtf32 tcgen05 update) + f64 refinement" if variant == "3xtf32" else \
        "f32 LU (ffma update) + f64 refinement"


FP64_PEAK_TF = 37.1   # measured: DFMA 36.9 / DMMA m8n8k4 37.1 TF/s on this pool's B200 (profiles/r02_ubench_fp64_peaks.txt)


def cusolver_context(dA, dB, reps: int = 2):
    """T3's "full double precision solve (reference time)" from the vendor library, for
    context only: cuSOLVER dgetrf + dgetrs through torch.linalg — never on the product path."""
    import torch
    Ac, Bc = dA.contiguous(), dB.contiguous()
    torch.linalg.lu_solve(*torch.linalg.lu_factor(Ac), Bc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        LU, piv = torch.linalg.lu_factor(Ac)
        torch.linalg.lu_solve(LU, piv, Bc)
    e1.record()
    torch.cuda.synchronize()
    del Ac
    return e0.elapsed_time(e1) / reps


def fp64_roofline(mp, dA, dB, nb):
    """One instrumented binary64 solve: its trailing update (DMMA) against the measured FP64 peak."""
    import torch
    _, info, rep = mp.mp_dgesv_ex(dA, dB, None, mp.make_opts(nb=nb, flags=2))
    torch.cuda.synchronize()
    k = rep.kernels().get("trail")
    if not k or k["ms"] <= 0:
        return None
    ach = k["work"] / (k["ms"] / 1e3) / 1e12
    la, sp, su = mp.mp_exec_info()
    return {"kernel": "binary64 trailing update (DMMA mma.sync m8n8k4 f64)", "bound": "fp64 pipe",
            "achieved": round(ach, 2), "peak": FP64_PEAK_TF, "unit": "TFLOP/s", "frac": round(ach / FP64_PEAK_TF, 4),
            "sms": su if la else 148, "frac_of_partition": round(ach / (FP64_PEAK_TF * (su if la else 148) / 148), 4),
            "peak_source": "measured, tools/ubench_fp64.cu"}


def time_solves(mp, dA, dB, opts, steps, fp64=False):
    import torch
    if fp64:
        mp.mp_dgesv_ex(dA, dB, None, opts, report=False)
    else:
        mp.mp_dsgesv_ex(dA, dB, None, opts, report=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = []
    e0.record()
    for _ in range(steps):
        if fp64:
            _, info, _ = mp.mp_dgesv_ex(dA, dB, None, opts, report=False)
            its.append(info)
        else:
            _, it, info, _ = mp.mp_dsgesv_ex(dA, dB, None, opts, report=False)
            its.append(it)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, its


def other_configs(mp, args, dev):
    """BASELINE.json's other configs (B:7-B:11), one or two solves each, reported beside the headline:
    C3 with the FFMA variant, C2, C4 (n = 49152, nrhs = 16, device-generated), C5 (kappa sweep)."""
    import torch
    res = {}
    # C3, FFMA variant (K5a), on the headline inputs
    A, B, _ = inputs.gaussian(args.n, nrhs=1, seed=inputs.BASE_SEED)
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    ms, its = time_solves(mp, dA, dB, mp.make_opts(variant=mp.MP_VARIANT_FFMA), 2)
    _, _, _, rep = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts(variant=mp.MP_VARIANT_FFMA, flags=2))
    torch.cuda.synchronize()
    t = rep.kernels().get("trail", {"ms": 0, "work": 0})
    ffma_peak = 148 * 128 * 2 * peaks()[0].get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    ach = t["work"] / (t["ms"] / 1e3) / 1e12 if t["ms"] else None
    res["C3_ffma"] = {"n": args.n, "variant": "ffma", "ms": round(ms, 3), "gflops": round(flops(args.n) / ms / 1e6, 1),
                      "iters": its, "trail_tflops": round(ach, 2) if ach else None,
                      "trail_frac_of_ffma_peak": round(ach / ffma_peak, 4) if ach else None,
                      "ffma_peak_tflops": round(ffma_peak, 1)}
    del dA, dB
    log("C2")
    # C2: n = 4096, nb = 128
    A, B, _ = inputs.gaussian(4096, nrhs=1, seed=inputs.BASE_SEED)
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    ms, its = time_solves(mp, dA, dB, mp.make_opts(nb=128), 5)
    ms64, _ = time_solves(mp, dA, dB, mp.make_opts(nb=128), 3, fp64=True)
    res["C2"] = {"n": 4096, "nb": 128, "ms": round(ms, 3), "gflops": round(flops(4096) / ms / 1e6, 1), "iters": its,
                 "fp64_ms": round(ms64, 3), "speedup_vs_fp64": round(ms64 / ms, 3)}
    log("C1")
    # C1: n = 512 (the paper: small n loses)
    A, B, _ = inputs.gaussian(512, nrhs=1, seed=inputs.BASE_SEED)
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    ms, its = time_solves(mp, dA, dB, mp.make_opts(nb=64), 10)
    ms64, _ = time_solves(mp, dA, dB, mp.make_opts(nb=64), 10, fp64=True)
    res["C1"] = {"n": 512, "nb": 64, "ms": round(ms, 3), "iters": its, "fp64_ms": round(ms64, 3),
                 "speedup_vs_fp64": round(ms64 / ms, 3)}
    log("C5")
    # C5: n = 8192, A = U diag(sigma) V^T, U, V from QR of Gaussian matrices (generated on the GPU here)
    n5 = 8192
    g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED + 2)
    U, _ = torch.linalg.qr(torch.randn((n5, n5), dtype=torch.float64, device=dev, generator=g))
    V, _ = torch.linalg.qr(torch.randn((n5, n5), dtype=torch.float64, device=dev, generator=g))
    xt = (torch.rand((1, n5), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
    c5 = []
    for kappa in (1e2, 1e4, 1e6, 1e8, 1e10):
        sig = kappa ** (-torch.arange(n5, dtype=torch.float64, device=dev) / (n5 - 1))
        Ak = ((U * sig[None, :]) @ V.t()).t().contiguous().t()       # column-major
        Bk = (Ak @ xt).t().contiguous().t()
        ms, its = time_solves(mp, Ak, Bk, mp.make_opts(), 2)
        c5.append({"kappa": kappa, "iters": its[0], "ms": round(ms, 3)})
        del Ak, Bk
    res["C5"] = {"n": n5, "sweep": c5, "note": "iters -31 = no convergence in 30 corrections, binary64 fallback "
                                                "(time includes the wasted refinement)"}
    del U, V
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    log("C4")
    # NEXT-4: extended-precision refinement (QDGESV analog) on the C3 inputs
    log("QD")
    A, B, _ = inputs.gaussian(args.n, nrhs=1, seed=inputs.BASE_SEED)
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    del A
    mp.mp_qdgesv_ex(dA, dB, report=False)
    torch.cuda.synchronize()
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record()
    _, _, itq, infoq, _ = mp.mp_qdgesv_ex(dA, dB, report=False)
    q1.record()
    torch.cuda.synchronize()
    _, _, _, _, repq = mp.mp_qdgesv_ex(dA, dB, opts=mp.make_opts(flags=2))
    torch.cuda.synchronize()
    kq = repq.kernels()
    rq = kq.get("residual", {"ms": 0, "work": 0})
    res["QD_C3"] = {"n": args.n, "what": "binary64 LU + double-double residual/update (stop at 2^-104)",
                    "ms": round(q0.elapsed_time(q1), 3), "iters": itq, "info": infoq,
                    "factor_ms": round(repq.t_factor_ms, 3), "refine_ms": round(repq.t_refine_ms, 3),
                    "dd_residual_gbs": round(rq["work"] / rq["ms"] / 1e6, 1) if rq["ms"] else None}
    del dA, dB
    # SPD variant (NEXT-1) at C3's size: A = G G^T / (2n), G n x 2n N(0,1), generated on the GPU
    log("SPD")
    ns = args.n
    g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED + 7)
    G = torch.randn((ns, 2 * ns), dtype=torch.float64, device=dev, generator=g)
    As = (G @ G.t()) / (2.0 * ns)
    del G
    As = 0.5 * (As + As.t())                                       # symmetric bytes; column-major = row-major
    xs = (torch.rand((1, ns), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
    Bs = (As @ xs).t().contiguous().t()
    Asc = As.t()                                                    # (n, n) stride (1, n) view
    mp.mp_dsposv_ex(Asc, Bs, None, mp.make_opts(), report=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = []
    for _ in range(3):
        _, it, _, _ = mp.mp_dsposv_ex(Asc, Bs, None, mp.make_opts(), report=False)
        its.append(it)
    e1.record()
    torch.cuda.synchronize()
    ms_s = e0.elapsed_time(e1) / 3
    _, it, _, rep = mp.mp_dsposv_ex(Asc, Bs, None, mp.make_opts(flags=2))
    torch.cuda.synchronize()
    kk = rep.kernels()
    mp.mp_dposv_ex(Asc, Bs, None, mp.make_opts(), report=False)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    mp.mp_dposv_ex(Asc, Bs, None, mp.make_opts(), report=False)
    f1.record()
    torch.cuda.synchronize()
    ms64 = f0.elapsed_time(f1)
    Ac = As.contiguous()
    torch.linalg.cholesky(Ac)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    Lc = torch.linalg.cholesky(Ac)
    torch.cholesky_solve(Bs.contiguous(), Lc)
    c1.record()
    torch.cuda.synchronize()
    tr = kk.get("trail", {"ms": 0, "work": 0})
    rr = kk.get("residual", {"ms": 0, "work": 0})
    spd_flops = ns ** 3 / 3.0
    res["SPD_C3"] = {"n": ns, "matrix": "Wishart G G^T/(2n), G n x 2n N(0,1) (kappa ~ 34)", "ms": round(ms_s, 3),
                     "gflops_n3_over_3": round(spd_flops / ms_s / 1e6, 1), "iters": its,
                     "factor_ms": round(rep.t_factor_ms, 3), "refine_ms": round(rep.t_refine_ms, 3),
                     "fp64_ms": round(ms64, 3), "speedup_vs_fp64": round(ms64 / ms_s, 3),
                     "cusolver_dpotrf_dpotrs_ms": round(c0.elapsed_time(c1), 3),
                     "syrk_tensor_tflops": round(3 * tr["work"] / tr["ms"] / 1e9, 1) if tr["ms"] else None,
                     "symv_residual_gbs": round(rr["work"] / rr["ms"] / 1e6, 1) if rr["ms"] else None,
                     "kernels_ms": {k: [round(v["ms"], 3), v["launches"]] for k, v in kk.items()}}
    del As, Ac, Lc, Bs, Asc
    torch.cuda.empty_cache()
    # Algorithm 2 (NEXT-3): FGMRES(10)-GMRES_SP(20) at C3's size on A = 2.5 I + G / sqrt(n)
    # (the stand-in for the paper's application matrices, inputs.shifted_gaussian), generated on the GPU
    log("FGMRES")
    g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED + 11)
    Ag = (torch.randn((ns, ns), dtype=torch.float64, device=dev, generator=g) / math.sqrt(ns)).t()
    Ag.diagonal().add_(2.5)
    xg = (torch.rand((1, ns), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
    bg = (Ag @ xg).t().contiguous().t()
    mp.mp_fgmres_ex(Ag, bg, m_out=10, m_in=20, report=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, itg, infog, _ = mp.mp_fgmres_ex(Ag, bg, m_out=10, m_in=20, report=False)
    e1.record()
    torch.cuda.synchronize()
    _, _, _, repg = mp.mp_fgmres_ex(Ag, bg, m_out=10, m_in=20, opts=mp.make_opts(flags=2))
    torch.cuda.synchronize()
    kg = repg.kernels()
    sg, rg = kg.get("solve", {"ms": 0, "work": 0}), kg.get("residual", {"ms": 0, "work": 0})
    ms_d, _ = time_solves(mp, Ag, bg, mp.make_opts(), 1)
    res["FGMRES_C3"] = {"n": ns, "m_out": 10, "m_in": 20, "matrix": "2.5 I + G/sqrt(n), G N(0,1)",
                        "ms": round(e0.elapsed_time(e1), 3), "outer_cycles": itg, "info": infog,
                        "launches": repg.kernel_launches,
                        "inner_cycle_gbs": round(sg["work"] / sg["ms"] / 1e6, 1) if sg["ms"] else None,
                        "outer_products_gbs": round(rg["work"] / rg["ms"] / 1e6, 1) if rg["ms"] else None,
                        "dsgesv_same_matrix_ms": round(ms_d, 3),
                        "kernels_ms": {k: [round(v["ms"], 3), v["launches"]] for k, v in kg.items()}}
    del Ag, bg, xg
    torch.cuda.empty_cache()
    # NEXT-2: the 1xTF32 factorisation (MP_VARIANT_TF32) with Algorithm 1 on a well-conditioned C3-sized
    # system (3 I + G / sqrt(n), kappa ~ 2), and with GMRES-IR (flags bit 8) on C3's Gaussian A itself
    log("TF32")
    g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED + 21)
    At = (torch.randn((ns, ns), dtype=torch.float64, device=dev, generator=g) / math.sqrt(ns)).t()
    At.diagonal().add_(3.0)
    xt = (torch.rand((1, ns), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
    bt = (At @ xt).t().contiguous().t()
    tf = {}
    for name, o in (("3xtf32", mp.make_opts()), ("tf32", mp.make_opts(variant=mp.MP_VARIANT_TF32))):
        ms_v, its_v = time_solves(mp, At, bt, o, 3)
        _, _, _, rep_v = mp.mp_dsgesv_ex(At, bt, None, o)
        torch.cuda.synchronize()
        tf[name] = {"ms": round(ms_v, 3), "iters": its_v, "factor_ms": round(rep_v.t_factor_ms, 3),
                    "refine_ms": round(rep_v.t_refine_ms, 3)}
    del At, bt, xt
    g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED)
    Ag = torch.randn((ns, ns), dtype=torch.float64, device=dev, generator=g).t()
    xg = (torch.rand((1, ns), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
    bg = (Ag @ xg).t().contiguous().t()
    gir = {}
    for name, o in (("tf32_alg1", mp.make_opts(variant=mp.MP_VARIANT_TF32)),
                    ("tf32_gmres_ir", mp.make_opts(variant=mp.MP_VARIANT_TF32, flags=256, itermax=63)),
                    ("3xtf32_gmres_ir", mp.make_opts(flags=256))):
        ms_v, its_v = time_solves(mp, Ag, bg, o, 1)
        _, _, _, rep_v = mp.mp_dsgesv_ex(Ag, bg, None, o)
        torch.cuda.synchronize()
        gir[name] = {"ms": round(ms_v, 3), "iters": its_v, "factor_ms": round(rep_v.t_factor_ms, 3),
                     "refine_ms": round(rep_v.t_refine_ms, 3), "fallback_ms": round(rep_v.t_fallback_ms, 3)}
    res["TF32_C3"] = {"n": ns, "well_conditioned": {"matrix": "3 I + G/sqrt(n) (kappa ~ 2)", **tf},
                      "gaussian": {"matrix": "C3's N(0,1) A", **gir}}
    del Ag, bg, xg
    torch.cuda.empty_cache()
    # C4: n = 49152, nrhs = 16 (A = 19.3 GB fp64), device-generated with a seeded torch generator
    if not args.no_c4:
        n4, r4 = 49152, 16
        g = torch.Generator(device=dev).manual_seed(inputs.BASE_SEED)
        dA = torch.randn((n4, n4), dtype=torch.float64, device=dev, generator=g).t()
        Xt = (torch.rand((r4, n4), dtype=torch.float64, device=dev, generator=g) * 2 - 1).t()
        dB = (dA @ Xt).t().contiguous().t()
        torch.cuda.synchronize()
        ms, its = time_solves(mp, dA, dB, mp.make_opts(), 1)
        _, _, _, rep = mp.mp_dsgesv_ex(dA, dB, None, mp.make_opts())
        torch.cuda.synchronize()
        ms64, _ = time_solves(mp, dA, dB, mp.make_opts(), 1, fp64=True)
        res["C4"] = {"n": n4, "nrhs": r4, "ms": round(ms, 1), "gflops": round(flops(n4) / ms / 1e6, 1), "iters": its,
                     "factor_ms": round(rep.t_factor_ms, 1), "refine_ms": round(rep.t_refine_ms, 1),
                     "fp64_ms": round(ms64, 1), "speedup_vs_fp64": round(ms64 / ms, 3)}
        # NEXT-2 at C4's size: 3 I + G / sqrt(n) (kappa ~ 2), 3xTF32 against the 1xTF32 factorisation
        dA.mul_(1.0 / math.sqrt(n4))
        dA.diagonal().add_(3.0)
        dB = (dA @ Xt).t().contiguous().t()
        torch.cuda.synchronize()
        tf4 = {}
        for name, o in (("3xtf32", mp.make_opts()), ("tf32", mp.make_opts(variant=mp.MP_VARIANT_TF32))):
            ms_v, its_v = time_solves(mp, dA, dB, o, 1)
            _, _, _, rep_v = mp.mp_dsgesv_ex(dA, dB, None, o)
            torch.cuda.synchronize()
            tf4[name] = {"ms": round(ms_v, 1), "iters": its_v, "factor_ms": round(rep_v.t_factor_ms, 1),
                         "refine_ms": round(rep_v.t_refine_ms, 1)}
        res["TF32_C4"] = {"n": n4, "nrhs": r4, "matrix": "3 I + G/sqrt(n) (kappa ~ 2)", **tf4}
        del dA, dB, Xt
        torch.cuda.empty_cache()
    return res


def log(msg: str):
    """Progress on stderr (the JSON line is the only stdout output)."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def main():
    import faulthandler
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--nb", type=int, default=0)
    ap.add_argument("--variant", default="3xtf32", choices=["ffma", "3xtf32"])
    ap.add_argument("--fp64-steps", type=int, default=2)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-n", type=int, default=8192)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C2/C4/C5/FFMA lines beside the headline")
    ap.add_argument("--no-c4", action="store_true", help="skip C4 (n = 49152) among the other configs")
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the 1D block-cyclic multi-GPU solver even at N = 1 (it is always used at N > 1)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", local if world > 1 else 0)

    from paper_0808_2794_b200 import binding as mp
    variant = mp.MP_VARIANT_FFMA if args.variant == "ffma" else mp.MP_VARIANT_3XTF32
    if world > 1 or args.dist:
        return run_distributed(args, rank, world, dev, dist, mp, variant)
    # timed region: CUDA events only around the trailing-update and residual launches (bit 3; a
    # handful per solve), resolved after the region (bit 2).  The full per-class breakdown comes
    # from one extra, untimed solve with events around every launch.
    opts = mp.make_opts(nb=args.nb, variant=variant, flags=2 | 4 | 8)
    n, nrhs = args.n, args.nrhs

    # inputs: one independent system per rank (weak scaling; replicas until the 1D block-cyclic path lands)
    A, B, Xt = inputs.gaussian(n, nrhs=nrhs, seed=inputs.BASE_SEED + rank)
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev).t()
    dB = torch.from_numpy(np.ascontiguousarray(B.T)).to(dev).t()
    dX = torch.empty((nrhs, n), dtype=torch.float64, device=dev).t()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def solve():
        _, it, info, rep = mp.mp_dsgesv_ex(dA, dB, dX, opts)
        return it, info, rep

    log("warm-up")
    clk = ClockSampler(dev.index).start()                         # running before the warm-up
    for _ in range(args.warmup):
        it, info, rep = solve()
    assert info == 0 and it >= 0, (it, info)
    mp.mp_profile_collect()                                         # drop the warm-up records

    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    barrier()
    torch.cuda.synchronize()
    walls = []
    with clk:
        e0.record(stream)
        for _ in range(args.steps):
            w0 = time.perf_counter()
            reps.append(solve())
            walls.append(time.perf_counter() - w0)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = flops(n) * args.steps * world / (ms_total / 1e3) / 1e9
    iters = [r[0] for r in reps]

    # trailing update + residual per-launch times over the timed region (CUDA events on the
    # launching stream); all other classes from one untimed fully instrumented solve
    kern = mp.mp_profile_collect().kernels()
    launches = sum(r[2].kernel_launches for r in reps)
    _, _, _, prep = mp.mp_dsgesv_ex(dA, dB, dX, mp.make_opts(nb=args.nb, variant=variant, flags=2))
    torch.cuda.synchronize()
    full = prep.kernels()
    for k, v in full.items():
        if k not in kern:
            kern[k] = {"ms": v["ms"] * args.steps, "work": v["work"] * args.steps, "launches": v["launches"] * args.steps}
    pk, pk_src = peaks()
    sm_max = pk.get("sm_max_mhz", 1965.0)
    ffma_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12           # TFLOP/s, FP32 FMA lanes x clock
    # TF32 tensor peak: the measured sustained bf16 cuBLAS figure x the nominal tf32/bf16 ratio (1.1 / 2.25)
    tf32_peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1400.0)) * (1.1 / 2.25)
    roof = None
    if "trail" in kern and kern["trail"]["ms"] > 0:
        # dominant contraction: the trailing Schur update A22 -= L21 U12; 3xTF32 does
        # 3 tensor-core products per useful product, so achieved = 3 x algorithmic flops / time
        d = kern["trail"]
        mult = 3.0 if args.variant == "3xtf32" else 1.0
        ach = mult * d["work"] / (d["ms"] / 1e3) / 1e12
        peak = tf32_peak if args.variant == "3xtf32" else ffma_peak
        la, sms_panel, sms_upd = mp.mp_exec_info()
        roof = {"kernel": "trailing Schur update (K5, %s)" % args.variant,
                "bound": "tensor" if args.variant == "3xtf32" else "alu",
                "achieved": round(ach, 2), "peak": round(peak, 1), "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                "traffic": _gemm_traffic() if args.variant == "3xtf32" else None,   # (the capture is of the 3xTF32 kernel)
                "peak_source": ("measured bf16_tflops_sustained x 1.1/2.25 (nominal tf32/bf16), " + pk_src)
                if args.variant == "3xtf32" else
                f"derived: 148 SM x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (sm_max_mhz, {pk_src})",
                "work_note": "achieved counts 3 x 2MNK tensor flops per launch for 3xTF32" if mult == 3.0 else "2MNK",
                "launches": d["launches"] // args.steps, "avg_launch_us": round(d["ms"] * 1e3 / d["launches"], 2),
                # with the look-ahead the update runs on a green context of sms_update SMs (the
                # panel keeps the rest): the same peak scaled to that partition
                "sms": sms_upd, "sms_total": 148,
                "frac_of_partition": round(ach / (peak * sms_upd / 148.0), 4)}
        alone = _gemm_alone(peak) if args.variant == "3xtf32" else None
        if alone:
            roof["alone_full_gpu"] = alone
    if "residual" in kern and kern["residual"]["ms"] > 0:
        d = kern["residual"]
        ach = d["work"] / (d["ms"] / 1e3) / 1e9
        roof_res = {"kernel": "residual r = b - A x (K8, fp64)", "bound": "hbm", "achieved": round(ach, 1),
                    "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(ach / pk["hbm_gbs"], 4),
                    "peak_source": pk_src}
    else:
        roof_res = None
    panel_us_col = None
    if "panel" in kern and kern["panel"]["launches"]:
        panel_us_col = round(kern["panel"]["ms"] * 1e3 / args.steps / n, 3)     # latency-bound: us per column
    breakdown = {k: {"ms_per_step": round(v["ms"] / args.steps, 3), "launches_per_step": v["launches"] // args.steps,
                     ("tflops" if k in ("gemm", "trsm", "panel", "trail") else "gbs"):
                         round(v["work"] / (v["ms"] / 1e3) / (1e12 if k in ("gemm", "trsm", "panel", "trail") else 1e9), 2)
                         if v["ms"] > 0 else None}
                 for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])}

    log("fp64 path")
    # FP64 path on the same inputs (speedup denominator, B:5)
    fp64_ms = None
    if args.fp64_steps > 0:
        o64 = mp.make_opts(nb=args.nb)
        Xd, info64, _ = mp.mp_dgesv_ex(dA, dB, None, o64)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.fp64_steps):
            mp.mp_dgesv_ex(dA, dB, Xd, o64, report=False)
        f1.record(stream)
        torch.cuda.synchronize()
        fp64_ms = f0.elapsed_time(f1) / args.fp64_steps
    log("fp64 roofline")
    roof64 = fp64_roofline(mp, dA, dB, args.nb) if args.fp64_steps > 0 else None
    log("cusolver context")
    cusolver_ms = cusolver_context(dA, dB) if args.fp64_steps > 0 else None

    log("e2e")
    # end-to-end through the C-ABI with pinned HOST buffers (copies inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        hA = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory()
        hB = torch.from_numpy(np.ascontiguousarray(B.T)).pin_memory()
        hX = torch.empty((nrhs, n), dtype=torch.float64).pin_memory()
        nA, nB, nX = hA.numpy().T, hB.numpy().T, hX.numpy().T      # Fortran views of pinned memory
        mp.mp_dsgesv_ex(nA, nB, nX, mp.make_opts(nb=args.nb, variant=variant), report=False)
        barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.e2e_steps):
            mp.mp_dsgesv_ex(nA, nB, nX, mp.make_opts(nb=args.nb, variant=variant), report=False)
        g1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = g0.elapsed_time(g1) / args.e2e_steps
        if dist is not None:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": round(flops(n) * world / (e2e_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 8 * n * n + 8 * n * nrhs, "d2h_bytes_per_step": 8 * n * nrhs,
               "ms_per_step": round(e2e_ms, 3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        dt, r, threads = cpu_oracle_sample(args.cpu_n, inputs.BASE_SEED)
        cpu = {"value": round(flops(args.cpu_n) / dt / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
               "kind": "oracle", "sample": f"one full oracle_dsgesv solve at n={args.cpu_n} (C3's generator at a "
                                           f"bounded size; GFLOP/s = 2n^3/3 of that n / its time: {dt:.1f} s, "
                                           f"iters={r.iters})"}
        import oracle
        nt = oracle.num_threads()
        oracle.set_num_threads(1)
        dt1, r1, _ = cpu_oracle_sample(512, inputs.BASE_SEED)
        oracle.set_num_threads(nt)
        cpu["c1_one_thread"] = {"n": 512, "s": round(dt1, 3), "gflops": round(flops(512) / dt1 / 1e9, 3),
                                "iters": r1.iters}
    log("other configs")
    extra = other_configs(mp, args, dev) if (rank == 0 and world == 1 and not args.no_configs) else None

    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(args.variant), "data": "synthetic",
               "config": {"workload": WORKLOAD, "n": n, "nrhs": nrhs, "nb": reps[-1][2].nb,
                          "variant": args.variant, "iters": iters,
                          "l2": "inputs larger than L2 (A fp64 = %.2f GB)" % (8 * n * n / 1e9),
                          "parallelism": "1 GPU" if world == 1 else f"{world} independent replicas",
                          "lookahead": "panel stream + %d-SM update green context" % mp.mp_exec_info()[2]
                          if mp.mp_exec_info()[0] else "off"},
               "speedup_vs_fp64": round(fp64_ms / ms_step, 3) if fp64_ms else None,
               "fp64_ms_per_step": round(fp64_ms, 3) if fp64_ms else None,
               "roofline_fp64_path": roof64,
               "fp64_context": {"cusolver_dgetrf_dgetrs_ms": round(cusolver_ms, 3),
                                "speedup_vs_cusolver": round(cusolver_ms / ms_step, 3),
                                "fp64_path_vs_cusolver": round(fp64_ms / cusolver_ms, 3) if fp64_ms else None,
                                "note": "vendor FP64 LU solve via torch.linalg (context only, not on the path)"}
               if cusolver_ms else None,
               "e2e": e2e, "roofline": roof, "roofline_residual": roof_res,
               "panel_us_per_column": panel_us_col, "kernels": breakdown, "cpu_baseline": cpu,
               "clocks": clk.summary(), "gpu_launches": launches, "other_configs": extra,
               "phases_ms": {"wall": round(1e3 * sum(walls) / len(walls), 3),
                             "call_device": round(sum(r[2].t_total_ms for r in reps) / len(reps), 3),
                             "demote": round(sum(r[2].t_demote_ms for r in reps) / len(reps), 3),
                             "factor": round(sum(r[2].t_factor_ms for r in reps) / len(reps), 3),
                             "refine": round(sum(r[2].t_refine_ms for r in reps) / len(reps), 3)}}
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
