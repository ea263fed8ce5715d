"""Parity of the CUDA path (through the C-ABI) against the CPU oracle (`-m gpu`).

Classes (= SURVEY.md §8(c)):
* EXACT   — constructed exact-LU family (pin P2): P, L, U, X bitwise, iters 0;
* STRICT  — prescribed-kappa inputs with parity budget B <= 1e-12:
            ||x_gpu - x_or||_inf / ||x_or||_inf <= 1e-12, |d iters| <= 1, both meet the criterion;
* CRITERION — Gaussian inputs: both meet the B:5 criterion (long-double certificate),
            |d iters| <= 1, forward error within the kappa bound; the x gap is reported;
* FALLBACK — kappa * eps_s > 1: both iters = -31, binary64 solutions agree.
Sizes span several tiles/blocks and ragged tails (n not a multiple of nb, of the
128-row solve block, of the 128x128 GEMM tile).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

pytestmark = pytest.mark.gpu

EPS32 = 2.0 ** -24
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


def perm_from_ipiv(ipiv):
    p = np.arange(len(ipiv))
    for k, q in enumerate(ipiv):
        p[k], p[q] = p[q], p[k]
    return p


def certificate_ok(A, X, B):
    """P9: long-double residual, B:5 criterion with its own ||A||_F."""
    n = A.shape[0]
    Al = np.asarray(A, dtype=np.longdouble)
    Xl = np.asarray(X, dtype=np.longdouble).reshape(n, -1)
    Bl = np.asarray(B, dtype=np.longdouble).reshape(n, -1)
    R = np.asarray(Bl - Al @ Xl, dtype=np.float64)
    anrm = float(np.sqrt(np.sum(Al * Al)))
    cte = anrm * EPS64 * math.sqrt(n)
    Xm = np.asarray(X).reshape(n, -1)
    for c in range(R.shape[1]):
        rn, xn = np.linalg.norm(R[:, c]), np.linalg.norm(Xm[:, c])
        if not (rn == 0.0 or rn < 1.05 * xn * cte):   # 5 %: the certificate's own rounding vs the fp64 residual
            return False
    return True


def gpu_solve(mp, A, B, **kw):
    import torch
    dA, dB = mp.colmajor_cuda(A), mp.colmajor_cuda(B)
    X, it, info, rep = mp.mp_dsgesv_ex(dA, dB, opts=mp.make_opts(**kw) if kw else None)
    torch.cuda.synchronize()
    return X.cpu().numpy().copy(order="F"), it, info, rep


# --------------------------------------------------------------------------- EXACT (P2)
@pytest.mark.parametrize("n,nb", [(1, 0), (7, 0), (64, 0), (200, 32), (513, 64), (1000, 0), (1536, 128), (1300, 384),
                                  (2100, 256)])
def test_exact_lu_factors_bitwise(mp, orc, n, nb):
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n)
    LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(nb=nb))
    assert info == 0
    assert np.array_equal(perm_from_ipiv(ipiv), perm)
    assert np.array_equal(np.tril(LU, -1).astype(np.float64), np.tril(L, -1))
    assert np.array_equal(np.triu(LU).astype(np.float64), U)
    LUo, ipivo, _ = orc.sgetf2(A)
    assert np.array_equal(ipiv, ipivo) and np.array_equal(LU, LUo)


@pytest.mark.parametrize("n,nrhs", [(64, 1), (513, 3), (1000, 16), (2100, 1)])
def test_exact_lu_solve_bitwise(mp, n, nrhs):
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=nrhs, seed=n + 1)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert (it, info) == (0, 0)
    assert np.array_equal(Xg, X)


def test_exact_lu_dgetrf_and_dgesv_bitwise(mp):
    A, B, X, perm, L, U = inputs.exact_lu(700, nrhs=2, seed=3)
    LU, ipiv, info = mp.mp_dgetrf(A)
    assert info == 0 and np.array_equal(perm_from_ipiv(ipiv), perm)
    assert np.array_equal(np.triu(LU), U) and np.array_equal(np.tril(LU, -1), np.tril(L, -1))
    import torch
    Xd, info, _ = mp.mp_dgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    assert info == 0 and np.array_equal(Xd.cpu().numpy(), X)


# --------------------------------------------------------------------------- STRICT
def parity_budget(n, kappa, A):
    return kappa * np.linalg.norm(A) * math.sqrt(n) * EPS64       # ||A||_2 = 1


@pytest.mark.parametrize("n,kappa,seed", [(512, 1.0, 0), (512, 2.0, 1), (1024, 1.0, 2), (1000, 10.0, 3),
                                          (1024, 2.0, 4), (256, 100.0, 0)])
def test_strict_parity(mp, orc, n, kappa, seed):
    A, B, X = inputs.conditioned(n, kappa, seed=seed)
    assert parity_budget(n, kappa, A) <= 1e-12
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert info == ro.info == 0
    assert it >= 0 and ro.iters >= 0 and abs(it - ro.iters) <= 1
    gap = np.abs(Xg - ro.X).max() / np.abs(ro.X).max()
    assert gap <= 1e-12, gap
    assert certificate_ok(A, Xg, B) and certificate_ok(A, ro.X, B)
    assert abs(rep.anrm - ro.anrm) <= 1e-13 * ro.anrm


# --------------------------------------------------------------------------- CRITERION
@pytest.mark.parametrize("n,nrhs,seed", [(512, 1, 0), (512, 1, 1), (512, 1, 2), (777, 2, 3), (1024, 1, 4),
                                         (1500, 5, 5)])
def test_criterion_parity_gaussian(mp, orc, n, nrhs, seed):
    A, B, X = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert info == ro.info == 0
    assert it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters, rep.history(), list(ro.hist))
    assert certificate_ok(A, Xg, B)
    kappa = np.linalg.cond(A)
    bound = kappa * np.linalg.norm(A) / np.linalg.norm(A, 2) * math.sqrt(n) * EPS64
    err = np.abs(Xg - X).max() / np.abs(X).max()
    assert err <= 4 * bound + 4 * kappa * EPS64
    # the residual-ratio history has the oracle's shape: > 1 until the last check
    h = rep.history()
    assert len(h) == it + 1 and h[-1] < 1.0 and all(v >= 1.0 for v in h[:-1])


# --------------------------------------------------------------------------- A-19 inverted diagonal blocks
@pytest.mark.parametrize("n,nrhs,seed", [(700, 1, 31), (1500, 3, 32), (2100, 16, 33), (1300, 6, 34)])
def test_solve_inv_vs_substitution(mp, orc, n, nrhs, seed):
    """Default solves (inverted 64x64 diagonal blocks) and plain substitution (flags bit 5)
    both reach the B:5 criterion within one iteration of the oracle."""
    A, B, X = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc.dsgesv(A, B)
    Xi, iti, infoi, repi = gpu_solve(mp, A, B)
    Xs, its, infos, reps = gpu_solve(mp, A, B, flags=32)
    assert repi.solve_inv == 1 and reps.solve_inv == 0
    assert infoi == infos == ro.info == 0
    assert abs(iti - ro.iters) <= 1 and abs(its - ro.iters) <= 1, (iti, its, ro.iters)
    assert certificate_ok(A, Xi, B) and certificate_ok(A, Xs, B)


@pytest.mark.parametrize("n,nrhs,seed", [(700, 20, 61), (1100, 33, 62), (600, 7, 63), (900, 2, 64)])
def test_many_rhs(mp, orc, n, nrhs, seed):
    """Several right-hand sides: the R = 4 / 8 / 16 sweep instantiations, and nrhs above one launch's
    16 columns (chunked sweeps, multi-column residual)."""
    A, B, X = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert info == ro.info == 0 and it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
    assert certificate_ok(A, Xg, B)


def block_kappa_max(L, U, bs=64):
    """max over the 64-row diagonal blocks of L and U of kappa_inf = ||T||_inf ||T^-1||_inf."""
    n = L.shape[0]
    k = 0.0
    for i0 in range(0, n, bs):
        for T in (L[i0:i0 + bs, i0:i0 + bs], U[i0:i0 + bs, i0:i0 + bs]):
            Ti = np.linalg.inv(T)
            k = max(k, np.abs(T).sum(1).max() * np.abs(Ti).sum(1).max())
    return k


@pytest.mark.parametrize("n,seed", [(300, 41), (513, 42)])
def test_solve_inv_gating(mp, n, seed):
    """The inverted blocks are used only when every diagonal block has kappa_inf <= 1e5
    (reading A-19); the exact-LU family (random dyadic triangles) stays on substitution
    and therefore exact."""
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=seed)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    expect = 1 if block_kappa_max(L, U) <= 1e5 else 0
    assert rep.solve_inv == expect
    assert info == 0 and certificate_ok(A, Xg, B)
    if expect == 0:
        assert it == 0 and np.array_equal(Xg, X)


def test_factor_parity_gaussian(mp, orc):
    n = 640
    A, _, _ = inputs.gaussian(n, seed=11)
    LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(nb=64))
    LUo, ipivo, _ = orc.sgetf2(A)
    assert info == 0
    diff = np.nonzero(ipiv != ipivo)[0]
    if diff.size:                                     # only a near-tie may flip a pivot
        k = diff[0]
        col = np.sort(np.abs(LUo[k:, k]))
        assert col[-1] - col[-2] <= 1e-4 * col[-1]
    else:
        rel = np.abs(LU.astype(np.float64) - LUo).max() / np.abs(LUo).max()
        assert rel <= 1e-4
    L = np.tril(LU, -1).astype(np.float64) + np.eye(n)
    U = np.triu(LU).astype(np.float64)
    PA = A.astype(np.float32).astype(np.float64)[perm_from_ipiv(ipiv), :]
    assert np.linalg.norm(PA - L @ U) / np.linalg.norm(A) <= 10 * n * EPS32
    assert np.abs(np.tril(LU, -1)).max() <= 1.0


@pytest.mark.parametrize("nb", [8, 32, 48, 96, 256, 320, 512])
def test_panel_width_invariance(mp, orc, nb):
    n = 900
    A, B, X = inputs.gaussian(n, nrhs=2, seed=21)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B, nb=nb)
    assert info == 0 and abs(it - ro.iters) <= 1 and certificate_ok(A, Xg, B)


# --------------------------------------------------------------------------- FALLBACK
@pytest.mark.parametrize("kappa", [1e10, 1e12])
def test_fallback_parity(mp, orc, kappa):
    n = 512
    A, B, X = inputs.conditioned(n, kappa, seed=7)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert (it, info) == (ro.iters, ro.info) == (-31, 0)
    gap = np.abs(Xg - ro.X).max() / np.abs(ro.X).max()
    assert gap <= kappa * math.sqrt(n) * EPS64 * 64
    R = np.asarray(B, np.longdouble) - np.asarray(A, np.longdouble) @ np.asarray(Xg, np.longdouble)
    assert np.linalg.norm(np.asarray(R, float)) <= 10 * n * EPS64 * np.linalg.norm(Xg)


def test_forced_fallback_and_dgesv(mp, orc):
    n = 600
    A, B, X = inputs.gaussian(n, nrhs=3, seed=5)
    Xg, it, info, rep = gpu_solve(mp, A, B, flags=1)
    assert (it, info) == (-31, 0)
    Xo, infoo = orc.dgesv(A, B)
    kappa = np.linalg.cond(A)
    assert np.abs(Xg - Xo).max() / np.abs(Xo).max() <= 8 * n * kappa * EPS64
    import torch
    Xd, infod, _ = mp.mp_dgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    assert infod == 0 and np.array_equal(Xd.cpu().numpy(), Xg)   # fallback == the mp_dgesv path


# --------------------------------------------------------------------------- edge cases
def test_edge_cases(mp, orc):
    # SPEC worked examples
    A = np.asfortranarray([[4.0, 3.0], [6.0, 3.0]])
    b = np.asfortranarray([[10.0], [12.0]])
    Xg, it, info, _ = gpu_solve(mp, A, b)
    assert info == 0 and np.allclose(Xg[:, 0], [1.0, 2.0], rtol=0, atol=1e-15)
    LU, ipiv, info = mp.mp_sgetrf(A)
    assert list(ipiv) == [1, 1] and LU[1, 0] == np.float32(2.0 / 3.0)
    # n = 1
    Xg, it, info, _ = gpu_solve(mp, np.asfortranarray([[3.0]]), np.asfortranarray([[6.0]]))
    assert (it, info) == (0, 0) and Xg[0, 0] == 2.0
    # b = 0 -> X = 0, iters 0 (A-3); A = I with fp32-representable b -> exact
    A, _, _ = inputs.gaussian(130, seed=1)
    Xg, it, info, _ = gpu_solve(mp, A, np.zeros((130, 2), order="F"))
    assert (it, info) == (0, 0) and not Xg.any()
    I = np.asfortranarray(np.eye(257))
    b = np.asfortranarray(np.arange(257, dtype=float)[:, None] / 8)
    Xg, it, info, _ = gpu_solve(mp, I, b)
    assert (it, info) == (0, 0) and np.array_equal(Xg, b)


def test_error_codes(mp, orc):
    A, B, X = inputs.gaussian(40, seed=4)
    A2 = A.copy(order="F"); A2[3, :] *= 1e39            # a row beyond FLT_MAX: demotion overflows
    B2 = np.asfortranarray(A2 @ X)
    Xg, it, info, _ = gpu_solve(mp, A2, B2)
    ro = orc.dsgesv(A2, B2)
    assert (it, info) == (ro.iters, ro.info) == (-2, 0)
    # FALLBACK class: the two binary64 solutions agree within the P8 bound
    # kappa (||A||_F / ||A||_2) sqrt(n) 2^-53, taken for the row-equilibrated matrix (= A: the
    # scaled row is A's row 3 times 1e39, and GEPP picks it first on both sides) — reading A-21
    kappa = np.linalg.cond(A)
    p8 = kappa * np.linalg.norm(A) / np.linalg.norm(A, 2) * math.sqrt(40) * EPS64
    assert np.abs(Xg - ro.X).max() <= p8 * np.abs(ro.X).max()
    assert np.abs(Xg - X).max() <= p8 * np.abs(X).max()
    Z = np.asfortranarray([[1.0, 1.0], [1.0, 1.0 + 1e-10]])
    zb = np.asfortranarray([[2.0], [2.0 + 1e-10]])
    Xg, it, info, _ = gpu_solve(mp, Z, zb)
    assert (it, info) == (-3, 0)
    S = np.asfortranarray([[1.0, 2.0], [2.0, 4.0]])
    Xg, it, info, _ = gpu_solve(mp, S, np.asfortranarray([[1.0], [2.0]]))
    assert (it, info) == (-3, 2)
    A3 = A.copy(order="F"); A3[0, 0] = np.nan
    assert gpu_solve(mp, A3, B)[2] == -3
    B3 = B.copy(order="F"); B3[1, 0] = np.inf
    assert gpu_solve(mp, A, B3)[2] == -5


def test_host_pointer_path_matches_device(mp):
    A, B, X = inputs.gaussian(1100, nrhs=2, seed=8)
    Xd, itd, infod, _ = gpu_solve(mp, A, B)
    Xh, ith, infoh, rep = mp.mp_dsgesv_ex(A, B)                 # numpy host buffers: staged by the library
    assert (ith, infoh) == (itd, infod) and np.array_equal(Xh, Xd)
    assert rep.t_copy_ms > 0


def test_deterministic(mp):
    A, B, X = inputs.gaussian(1300, nrhs=1, seed=9)
    X1 = gpu_solve(mp, A, B)[0]
    X2 = gpu_solve(mp, A, B)[0]
    assert np.array_equal(X1, X2)


def test_lda_larger_than_n(mp, orc):
    n, lda = 333, 350
    A, B, X = inputs.gaussian(n, seed=12)
    big = np.zeros((lda, n), order="F")
    big[:n, :] = A
    import torch
    dA = mp.colmajor_cuda(big)[:n, :]                             # view with stride (1, lda)
    assert dA.stride() == (1, lda)
    Xg, it, info, _ = mp.mp_dsgesv_ex(dA, mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    assert info == 0 and certificate_ok(A, Xg.cpu().numpy(), B)


# --------------------------------------------------------------------------- 3xTF32 tcgen05 variant (B:5)
@pytest.mark.parametrize("n", [700, 2100])
def test_exact_lu_factors_bitwise_3xtf32(mp, orc, n):
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n + 5)
    LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(variant=mp.MP_VARIANT_3XTF32))
    assert info == 0
    assert np.array_equal(perm_from_ipiv(ipiv), perm)
    assert np.array_equal(np.tril(LU, -1).astype(np.float64), np.tril(L, -1))
    assert np.array_equal(np.triu(LU).astype(np.float64), U)
    Xg, it, info, _ = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_3XTF32)
    assert (it, info) == (0, 0) and np.array_equal(Xg, X)


@pytest.mark.parametrize("n,nrhs,seed", [(1024, 1, 4), (1500, 5, 5), (2600, 1, 6)])
def test_criterion_parity_3xtf32(mp, orc, n, nrhs, seed):
    A, B, X = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_3XTF32)
    assert info == ro.info == 0
    assert it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters, rep.history(), list(ro.hist))
    assert certificate_ok(A, Xg, B)


def test_strict_parity_3xtf32(mp, orc):
    A, B, X = inputs.conditioned(1024, 1.0, seed=2)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_3XTF32)
    assert info == 0 and abs(it - ro.iters) <= 1
    assert np.abs(Xg - ro.X).max() / np.abs(ro.X).max() <= 1e-12


# --------------------------------------------------------------------------- FFMA variant (B:5), explicitly
# (the library default is the 3xTF32 variant; the tests above without options exercise it)
@pytest.mark.parametrize("n", [700, 2100])
def test_exact_lu_factors_bitwise_ffma(mp, orc, n):
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n + 7)
    LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(variant=mp.MP_VARIANT_FFMA))
    assert info == 0
    assert np.array_equal(perm_from_ipiv(ipiv), perm)
    assert np.array_equal(np.tril(LU, -1).astype(np.float64), np.tril(L, -1))
    assert np.array_equal(np.triu(LU).astype(np.float64), U)
    Xg, it, info, _ = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_FFMA)
    assert (it, info) == (0, 0) and np.array_equal(Xg, X)


@pytest.mark.parametrize("n,nrhs,seed", [(1024, 1, 4), (2600, 3, 6)])
def test_criterion_parity_ffma(mp, orc, n, nrhs, seed):
    A, B, X = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_FFMA)
    assert info == ro.info == 0
    assert it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters, rep.history(), list(ro.hist))
    assert certificate_ok(A, Xg, B)


def test_strict_parity_ffma(mp, orc):
    A, B, X = inputs.conditioned(1024, 1.0, seed=3)
    ro = orc.dsgesv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_FFMA)
    assert info == 0 and abs(it - ro.iters) <= 1
    assert np.abs(Xg - ro.X).max() / np.abs(ro.X).max() <= 1e-12


_EXCHANGE_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_0808_2794_b200 import binding as mp, inputs
n, nrhs, seed = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
A, B, _ = inputs.gaussian(n, nrhs=nrhs, seed=seed)
X, it, info, rep = mp.mp_dsgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
torch.cuda.synchronize()
np.save(sys.argv[5], X.cpu().numpy())
print(it, info)
"""


@pytest.mark.parametrize("n,nrhs,seed", [(1500, 3, 71), (700, 20, 72), (1200, 6, 73)])
def test_solve_exchange_modes_bitwise(mp, tmp_path, n, nrhs, seed):
    """The tagged {value, tag} y/F exchange of the binary32 sweeps and the epoch-flag exchange
    (MP_SOLVE_FLAGS=1, read once per process: run in a child) move the same values, so the
    whole solve is bitwise identical."""
    import os
    import subprocess
    import sys
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    A, B, _ = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    X, it, info, rep = mp.mp_dsgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    Xt = X.cpu().numpy()
    out = str(tmp_path / "x_flags.npy")
    env = dict(os.environ, MP_SOLVE_FLAGS="1")
    r = subprocess.run([sys.executable, "-c", _EXCHANGE_CHILD, root, str(n), str(nrhs), str(seed), out],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    it_f, info_f = map(int, r.stdout.split()[-2:])
    assert info == info_f == 0 and it == it_f
    assert np.array_equal(Xt.view(np.uint64), np.load(out).view(np.uint64))


_LL_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_0808_2794_b200 import binding as mp, inputs
import oracle
n = int(sys.argv[2])
A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n)
LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(nb=256))
p = np.arange(n)
for k, q in enumerate(ipiv):
    p[k], p[q] = p[q], p[k]
ok = info == 0 and np.array_equal(p, perm) and np.array_equal(np.tril(LU, -1).astype(float), np.tril(L, -1)) \
     and np.array_equal(np.triu(LU).astype(float), U)
A2, B2, _ = inputs.gaussian(n, nrhs=2, seed=n + 1)
ro = oracle.dsgesv(A2, B2)
Xg, it, info2, _ = mp.mp_dsgesv_ex(mp.colmajor_cuda(A2), mp.colmajor_cuda(B2))
torch.cuda.synchronize()
print(int(ok), it, ro.iters, info2)
"""


@pytest.mark.parametrize("n", [700, 2100])
def test_left_looking_panel_option(mp, n):
    """The experimental left-looking leaves (MP_PANEL_LL=1, read once per process: run in a child)
    reproduce the exact-LU factors bitwise and refine Gaussian systems within one iteration of the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _LL_CHILD, root, str(n)], env=dict(os.environ, MP_PANEL_LL="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ok, it, it_or, info = map(int, r.stdout.split()[-4:])
    assert ok == 1 and info == 0 and abs(it - it_or) <= 1


_CLUSTER_CHILD = """
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_0808_2794_b200 import binding as mp, inputs
n = int(sys.argv[2])
A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n)
LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(nb=256))
p = np.arange(n)
for k, q in enumerate(ipiv):
    p[k], p[q] = p[q], p[k]
ok = info == 0 and np.array_equal(p, perm) and np.array_equal(np.tril(LU, -1).astype(float), np.tril(L, -1)) \
     and np.array_equal(np.triu(LU).astype(float), U)
Ac, Bc, Xc, Lc = inputs.exact_chol(n, nrhs=1, seed=n + 17)
Lg, infoc = mp.mp_spotrf(Ac, mp.make_opts(nb=256))
ok = ok and infoc == 0 and np.array_equal(np.tril(Lg).astype(np.float64), Lc)
h = hashlib.sha1()
A2, B2, _ = inputs.gaussian(n, nrhs=2, seed=n + 1)
Xg, it, info2, _ = mp.mp_dsgesv_ex(mp.colmajor_cuda(A2), mp.colmajor_cuda(B2))
torch.cuda.synchronize()
h.update(Xg.cpu().numpy().tobytes())
LU2, ipiv2, info3 = mp.mp_sgetrf(A2, mp.make_opts(nb=128))
h.update(np.ascontiguousarray(LU2).tobytes()); h.update(np.ascontiguousarray(ipiv2).tobytes())
A3, B3, _ = inputs.spd_wishart(n, nrhs=1, seed=n + 2)
X3, it3, info4, _ = mp.mp_dsposv_ex(mp.colmajor_cuda(A3), mp.colmajor_cuda(B3))
torch.cuda.synchronize()
h.update(X3.cpu().numpy().tobytes())
print(int(ok), it, it3, info2 + info3 + info4, h.hexdigest())
"""


@pytest.mark.parametrize("n", [1300, 2600])
def test_update_cluster_modes_bitwise(mp, n):
    """The tensor-core update's cluster modes (MP_GEMM_CLUSTER, read once per process: run in children
    with MP_GEMM_CLUSTER_WAVES=0 so that every tcgen05 launch takes the mode, whatever its size): CTA
    pairs (8, tcgen05 cta_group::2, the default for large launches) and multicast clusters (2, 4) give
    the exact-LU / exact-Cholesky factors bitwise and the same bits as single CTAs (1) for Gaussian
    LU factors, the refined solution and the SPD solve (LOWER tiles: a pair's tile above the diagonal
    stores nothing)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for cs in (1, 2, 4, 8):
        r = subprocess.run([sys.executable, "-c", _CLUSTER_CHILD, root, str(n)],
                           env=dict(os.environ, MP_GEMM_CLUSTER=str(cs), MP_GEMM_CLUSTER_WAVES="0"),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[cs] = r.stdout.split()[-5:]
        assert res[cs][0] == "1" and res[cs][3] == "0", (cs, res[cs])
    assert res[2] == res[1] and res[4] == res[1] and res[8] == res[1], res
