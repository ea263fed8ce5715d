"""Parity at the configs BASELINE.json names (B:7-B:11), in the launch configuration bench.py times
(`-m gpu`).  These are the sizes where the factorisation picks its large leaf-cluster
configurations (9-16-CTA non-portable clusters, 256 x 4 leaves for m > 8192, the m > 16384 leaf
instantiations at C4) — the small-size suite in test_gpu_parity.py never reaches them.

* C2  n = 4096, nb = 128 Gaussian          — CRITERION: both meet B:5's test (long-double
                                              certificate P9), |d iters| <= 1; x gap reported
* C3  n = 16384, nb = 256 Gaussian, seed 2794 (the bench input) — CRITERION
* C5  n = 8192, kappa in {1e2, 1e4, 1e6}   — CRITERION + forward error within the P8 bound
      kappa in {1e8, 1e10}                 — FALLBACK: both -31, binary64 solutions agree
* STRICT kappa = 1 at n = 2048 / 4096 (parity budget n 2^-53 <= 1e-12): x gap <= 1e-12;
      n = 8192 (budget 9.1e-13, at the tolerance itself): 1e-12 when both sides stop at the same
      correction, else the rigorous stop bound of reading A-20
* EXACT  constructed exact-LU family (pin P2) at n = 4096, 16384 and 49152 (C4's size):
      P, L, U and X bitwise, iters 0 — no oracle needed, the answer is known by construction.

Results (iterations, gaps, times) are appended as JSON lines to $MP_PARITY_LOG when it is set.
"""
from __future__ import annotations

import json
import math
import os
import time

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

pytestmark = pytest.mark.gpu

EPS64 = 2.0 ** -53


@pytest.fixture(scope="module")
def mp():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0808_2794_b200 import build
    build.build()
    from paper_0808_2794_b200 import binding
    return binding


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def log(rec):
    path = os.environ.get("MP_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


def residual_ld(A, X, B, chunk=1024):
    """b - A x with long-double accumulation (P9), by column chunks so n = 16384 stays in memory."""
    n = A.shape[0]
    Xl = np.asarray(X, np.longdouble).reshape(n, -1)
    R = np.asarray(B, np.longdouble).reshape(n, -1).copy()
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        R -= np.asarray(A[:, j0:j1], np.longdouble) @ Xl[j0:j1]
    return np.asarray(R, np.float64)


def certificate(A, X, B):
    """max over columns of ||r|| / (||x|| ||A||_F 2^-53 sqrt(n)) with the long-double residual."""
    n = A.shape[0]
    R = residual_ld(A, X, B)
    anrm = math.sqrt(sum(float(np.sum(np.asarray(A[:, j0:j0 + 2048], np.longdouble) ** 2))
                         for j0 in range(0, n, 2048)))
    cte = anrm * EPS64 * math.sqrt(n)
    Xm = np.asarray(X).reshape(n, -1)
    worst = 0.0
    for c in range(R.shape[1]):
        rn, xn = np.linalg.norm(R[:, c]), np.linalg.norm(Xm[:, c])
        worst = max(worst, 0.0 if rn == 0.0 else rn / (xn * cte))
    return worst


def gpu_solve(mp, A, B, **kw):
    import torch
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    t0 = time.perf_counter()
    X, it, info, rep = mp.mp_dsgesv_ex(dA, dB, opts=mp.make_opts(**kw) if kw else None)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    del dA
    return X.cpu().numpy().copy(order="F"), it, info, rep, dt


def oracle_solve(orc, A, B):
    t0 = time.perf_counter()
    ro = orc.dsgesv(A, B)
    return ro, time.perf_counter() - t0


def check_criterion(cfg, mp, orc, A, B, Xtrue, nb=0, kappa=None):
    Xg, it, info, rep, tg = gpu_solve(mp, A, B, nb=nb)
    ro, to = oracle_solve(orc, A, B)
    cg, co = certificate(A, Xg, B), certificate(A, ro.X, B)
    gap = float(np.abs(Xg - ro.X).max() / np.abs(ro.X).max())
    ferr = float(np.abs(Xg - Xtrue).max() / np.abs(Xtrue).max())
    log({"cfg": cfg, "n": A.shape[0], "kappa": kappa, "iters_gpu": it, "iters_oracle": ro.iters,
         "info": [info, ro.info], "x_gap": gap, "fwd_err_gpu": ferr, "cert_gpu": cg, "cert_oracle": co,
         "hist_gpu": rep.history(), "hist_oracle": list(map(float, ro.hist)), "t_gpu_s": tg, "t_oracle_s": to})
    assert info == ro.info == 0
    assert it >= 0 and ro.iters >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
    assert cg < 1.05 and co < 1.05, (cg, co)           # both meet B:5's test (5 %: certificate rounding)
    assert abs(rep.anrm - ro.anrm) <= 1e-12 * ro.anrm
    return Xg, ro, gap, ferr


# --------------------------------------------------------------------------- C2, C3 (Gaussian)
def test_c2_n4096_criterion(mp, orc):
    A, B, X = inputs.gaussian(4096, nrhs=1, seed=inputs.BASE_SEED)
    check_criterion("C2", mp, orc, A, B, X, nb=128)


def test_c3_n16384_criterion(mp, orc):
    """The bench input itself (seed 2794, nb 256, default 3xTF32 variant, look-ahead on)."""
    A, B, X = inputs.gaussian(16384, nrhs=1, seed=inputs.BASE_SEED)
    check_criterion("C3", mp, orc, A, B, X, nb=256)


# --------------------------------------------------------------------------- C5 (conditioning sweep)
@pytest.fixture(scope="module")
def uv8192():
    n = 8192
    return (inputs.haar_orthogonal(n, inputs.BASE_SEED + 2), inputs.haar_orthogonal(n, inputs.BASE_SEED + 3))


def p8_bound(A, kappa):
    """B(A) = kappa (||A||_F / ||A||_2) sqrt(n) 2^-53 with ||A||_2 = 1 by construction."""
    n = A.shape[0]
    return kappa * np.linalg.norm(A) * math.sqrt(n) * EPS64


@pytest.mark.parametrize("kappa", [1e2, 1e4, 1e6])
def test_c5_criterion(mp, orc, uv8192, kappa):
    A, B, X = inputs.conditioned(8192, kappa, seed=inputs.BASE_SEED, UV=uv8192)
    Xg, ro, gap, ferr = check_criterion("C5", mp, orc, A, B, X, nb=256, kappa=kappa)
    bound = p8_bound(A, kappa)
    assert ferr <= bound, (ferr, bound)
    assert np.abs(ro.X - X).max() / np.abs(X).max() <= bound


@pytest.mark.parametrize("kappa", [1e8, 1e10])
def test_c5_fallback(mp, orc, uv8192, kappa):
    """kappa eps_s > 1: refinement cannot converge; both sides hit the 30 cap and
    solve in binary64.  The two binary64 GEPP solutions agree within the P8 bound."""
    A, B, X = inputs.conditioned(8192, kappa, seed=inputs.BASE_SEED, UV=uv8192)
    Xg, it, info, rep, tg = gpu_solve(mp, A, B, nb=256)
    ro, to = oracle_solve(orc, A, B)
    gap = float(np.abs(Xg - ro.X).max() / np.abs(ro.X).max())
    R = residual_ld(A, Xg, B)
    bwd = float(np.linalg.norm(R) / (np.linalg.norm(A) * np.linalg.norm(Xg)))
    log({"cfg": "C5", "n": 8192, "kappa": kappa, "iters_gpu": it, "iters_oracle": ro.iters,
         "info": [info, ro.info], "x_gap": gap, "bwd_err_gpu": bwd, "t_gpu_s": tg, "t_oracle_s": to})
    assert (it, info) == (ro.iters, ro.info) == (-31, 0)
    assert gap <= p8_bound(A, kappa)
    assert bwd <= 8192 * EPS64


# --------------------------------------------------------------------------- STRICT at size
@pytest.mark.parametrize("n", [2048, 4096])
def test_strict_kappa1(mp, orc, n):
    A, B, X = inputs.conditioned(n, 1.0, seed=n)
    assert p8_bound(A, 1.0) <= 1e-12
    Xg, ro, gap, ferr = check_criterion("STRICT", mp, orc, A, B, X, kappa=1.0)
    assert gap <= 1e-12, gap


def stop_bound(A, X, ratio, kappa):
    """Forward error any iterate passing B:5's test can have (reading A-20): with ||A||_2 = 1 and
    ||A^-1||_2 = kappa (C5 generator), ||x - x*||_inf <= ||x - x*||_2 <= kappa ||r||_2
    < kappa * ratio * ||x||_2 ||A||_F sqrt(n) 2^-53."""
    n = A.shape[0]
    return kappa * ratio * np.linalg.norm(X) * np.linalg.norm(A) * math.sqrt(n) * EPS64


def test_kappa1_8192_budget_edge(mp, orc, uv8192):
    """kappa = 1 at n = 8192: the parity budget n 2^-53 = 9.1e-13 sits at the 1e-12 tolerance itself,
    so B:5's own stop test admits iterates 1e-12 apart (reading A-20).  When both sides stop at the
    same correction the STRICT 1e-12 gap is required; when they stop one correction apart (allowed,
    |d iters| <= 1) the gap must lie within the sum of the two stop bounds above."""
    A, B, X = inputs.conditioned(8192, 1.0, seed=inputs.BASE_SEED, UV=uv8192)
    Xg, ro, gap, ferr = check_criterion("STRICT-edge", mp, orc, A, B, X, kappa=1.0)
    _, it_g, _, rep, _ = gpu_solve(mp, A, B)            # deterministic: the same solve again, for its report
    if it_g == ro.iters:
        assert gap <= 1e-12, gap
    else:
        bound = (stop_bound(A, Xg, rep.history()[-1], 1.0) + stop_bound(A, ro.X, float(ro.hist[-1]), 1.0))
        assert gap <= bound / np.abs(ro.X).max(), (gap, bound)


# --------------------------------------------------------------------------- EXACT (P2) at size
def _exact_case(mp, n, nb, variant, solve, fp64=False):
    import ctypes
    import torch
    A, B, X, perm, L, U = inputs.exact_lu_device(n, nrhs=2, seed=n + variant)
    torch.cuda.synchronize()
    LU = torch.empty((n, n), dtype=torch.float64 if fp64 else torch.float32, device="cuda")   # column-major
    ipiv = torch.empty(n, dtype=torch.int32, device="cuda")
    info = ctypes.c_int(7)
    opts = mp.make_opts(nb=nb, variant=variant)
    mp.lib.mp_set_stream(torch.cuda.current_stream().cuda_stream)
    t0 = time.perf_counter()
    getrf = mp.lib.mp_dgetrf if fp64 else mp.lib.mp_sgetrf
    mp._check(getrf(n, A.data_ptr(), n, LU.data_ptr(), ipiv.data_ptr(), ctypes.byref(info), ctypes.byref(opts)))
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    assert info.value == 0
    LUr = LU.view(n, n)                     # LUr[j, i] = LU(i, j)  (column-major buffer read row-major)
    # L strictly below the diagonal, U on and above, bitwise
    Lg = torch.tril(LUr.t(), -1)
    ok_l = torch.equal(Lg, torch.tril(L, -1).to(LUr.dtype))
    del Lg
    ok_u = torch.equal(torch.triu(LUr.t()), U.to(LUr.dtype))
    del LU, LUr
    # pivots: replay the sequential interchanges into a permutation
    ip = ipiv.cpu().numpy()
    p = np.arange(n)
    for k, q in enumerate(ip):
        p[k], p[q] = p[q], p[k]
    ok_p = np.array_equal(p, perm.cpu().numpy())
    rec = {"cfg": "EXACT", "n": n, "nb": nb, "variant": "fp64" if fp64 else variant, "P": ok_p, "L": ok_l,
           "U": ok_u, "t_getrf_s": tf}
    if solve and fp64:
        Xg, info2, rep = mp.mp_dgesv_ex(A, B, opts=opts)
        torch.cuda.synchronize()
        it = 0
        rec.update(info=info2, X=bool(torch.equal(Xg, X)))
    elif solve:
        Xg, it, info2, rep = mp.mp_dsgesv_ex(A, B, opts=opts)
        torch.cuda.synchronize()
        rec.update(iters=it, info=info2, X=bool(torch.equal(Xg, X)))
    log(rec)
    assert ok_p and ok_l and ok_u
    if solve:
        assert (it, info2) == (0, 0) and rec["X"]


@pytest.mark.parametrize("variant", [0, 1])
def test_exact_lu_4096(mp, variant):
    _exact_case(mp, 4096, 128, variant, True)


def test_exact_lu_16384(mp):
    _exact_case(mp, 16384, 256, 1, True)


def test_exact_lu_49152(mp):
    """C4's size: the m > 16384 leaf instantiations and the largest clusters."""
    _exact_case(mp, 49152, 256, 1, True)


def test_exact_lu_fp64_36864(mp):
    """The binary64 path (mp_dgetrf / mp_dgesv, the fallback) above 32768 rows, where its leaves are
    4 columns wide (512 x 8 rows per CTA, 16-CTA cluster): P, L, U and X bitwise."""
    _exact_case(mp, 36864, 256, 1, True, fp64=True)


def test_streamed_host_path_exact_and_criterion(mp, orc):
    """Host buffers (the end-to-end path) with n >= 4096: A crosses PCIe in column blocks while the
    factorisation runs.  The exact-LU family stays bitwise (iters 0, X = x_true) and a
    Gaussian system gives the device path's result bitwise (same operations, reordered only across
    independent column blocks)."""
    import torch
    n = 4608
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n)
    Xh, it, info, rep = mp.mp_dsgesv_ex(A, B)
    assert (it, info) == (0, 0) and np.array_equal(Xh, X)
    A2, B2, _ = inputs.gaussian(n, nrhs=2, seed=77)
    Xh2, ith, infoh, reph = mp.mp_dsgesv_ex(A2, B2)
    Xd2, itd, infod, repd, _ = gpu_solve(mp, A2, B2)
    ro = orc.dsgesv(A2, B2)
    log({"cfg": "streamed-host", "n": n, "iters_host": ith, "iters_dev": itd, "iters_oracle": ro.iters,
         "x_gap_host_dev": float(np.abs(Xh2 - Xd2).max() / np.abs(Xd2).max()),
         "anrm_rel": abs(reph.anrm - ro.anrm) / ro.anrm})
    assert infoh == infod == 0 and abs(ith - ro.iters) <= 1
    assert certificate(A2, Xh2, B2) < 1.05
    assert abs(reph.anrm - ro.anrm) <= 1e-12 * ro.anrm


_STREAM_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_0808_2794_b200 import binding as mp, inputs
n = int(sys.argv[2])
A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n)
Xh, it, info, _ = mp.mp_dsgesv_ex(A, B)
ok = int(it == 0 and info == 0 and np.array_equal(Xh, X))
A2, B2, _ = inputs.gaussian(n, nrhs=2, seed=77)
Xh2, ith, infoh, _ = mp.mp_dsgesv_ex(A2, B2)
Xd2, itd, infod, _ = mp.mp_dsgesv_ex(mp.colmajor_cuda(A2), mp.colmajor_cuda(B2))
torch.cuda.synchronize()
same = int(infoh == infod == 0 and ith == itd and np.array_equal(Xh2, Xd2.cpu().numpy()))
print(ok, same)
"""


@pytest.mark.parametrize("env", [{"MP_STREAM_JOINED": "1"}, {"MP_STREAM_JOINED": "1", "MP_STREAM_PLAN": "2,3,1,4,2,1"},
                                 {"MP_H2D_SM": "1"}])
def test_streamed_host_path_options(env):
    """The streamed e2e path's experimental options (read once per process: run in a child): blocks
    joining one look-ahead loop (interchanges reach a block from its join on, catch-up spread over the
    steps) and the SM-load copy of the host blocks.  Exact-LU stays bitwise and the Gaussian solve
    equals the device-resident path bitwise (the same operations per entry)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _STREAM_CHILD, root, "4608"], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ok, same = map(int, r.stdout.split()[-2:])
    assert ok == 1 and same == 1
