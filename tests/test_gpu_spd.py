"""Parity of the SPD variant (P:369-371 SPOTRF / SPOTRS / DSYMM) through the C-ABI
against the CPU oracle (oracle/oracle_chol.c), `-m gpu`.

Classes as for the nonsymmetric path: EXACT (constructed exact-Cholesky family: L bitwise,
X bitwise with substitution solves), STRICT (kappa = 1: x gap <= 1e-12), CRITERION (both meet B:5's test
with the long-double certificate, |d iters| <= 1), FALLBACK (kappa eps_s > 1: both hand over to the
binary64 Cholesky, whose solutions agree within the P8 bound).  Sizes span several 256 / 128 panels,
ragged tails and the 3xTF32 SYRK tile grid (256 x 128 tiles, lower tiles only)."""
from __future__ import annotations

import math

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


def certificate(A, X, B):
    n = A.shape[0]
    Al = np.asarray(A, np.longdouble)
    R = np.asarray(np.asarray(B, np.longdouble).reshape(n, -1) - Al @ np.asarray(X, np.longdouble).reshape(n, -1),
                   np.float64)
    cte = float(np.sqrt(np.sum(Al * Al))) * EPS64 * math.sqrt(n)
    Xm = np.asarray(X).reshape(n, -1)
    return max(0.0 if np.linalg.norm(R[:, c]) == 0 else np.linalg.norm(R[:, c]) / (np.linalg.norm(Xm[:, c]) * cte)
               for c in range(R.shape[1]))


def gpu_solve(mp, A, B, **kw):
    import torch
    X, it, info, rep = mp.mp_dsposv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B), opts=mp.make_opts(**kw) if kw else None)
    torch.cuda.synchronize()
    return X.cpu().numpy().copy(order="F"), it, info, rep


# ------------------------------------------------------------------------- EXACT
@pytest.mark.parametrize("n,nb,variant", [(1, 0, 1), (7, 0, 1), (64, 0, 1), (300, 64, 1), (1000, 0, 1),
                                          (2100, 256, 1), (2100, 256, 0), (1300, 128, 0)])
def test_exact_cholesky_factor_bitwise(mp, orc, n, nb, variant):
    A, B, X, L = inputs.exact_chol(n, nrhs=1, seed=n + 17)
    Lg, info = mp.mp_spotrf(A, mp.make_opts(nb=nb, variant=variant))
    assert info == 0
    assert np.array_equal(np.tril(Lg).astype(np.float64), L)
    Lo, info_o = orc.spotf2(A)
    assert info_o == 0 and np.array_equal(np.tril(Lg), np.tril(Lo))


@pytest.mark.parametrize("n", [200, 700, 1500])
def test_exact_cholesky_fp64_factor_bitwise(mp, n):
    A, B, X, L = inputs.exact_chol(n, nrhs=1, seed=n + 19)
    Lg, info = mp.mp_dpotrf(A)
    assert info == 0 and np.array_equal(np.tril(Lg), L)


@pytest.mark.parametrize("n,nrhs", [(64, 1), (513, 3), (1400, 2)])
def test_exact_cholesky_solve_bitwise(mp, n, nrhs):
    """Substitution solves (flags bit 5) keep the exact family exact: iters 0, X == x_true bitwise.
    The binary64 path too."""
    import torch
    A, B, X, L = inputs.exact_chol(n, nrhs=nrhs, seed=n + 23)
    Xg, it, info, rep = gpu_solve(mp, A, B, flags=32)
    assert (it, info) == (0, 0) and np.array_equal(Xg, X)
    Xd, infod, _ = mp.mp_dposv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    assert infod == 0 and np.array_equal(Xd.cpu().numpy(), X)


# ------------------------------------------------------------------------- STRICT / CRITERION
@pytest.mark.parametrize("n,seed", [(512, 0), (1024, 1)])
def test_strict_spd_kappa1(mp, orc, n, seed):
    A, B, X = inputs.spd_conditioned(n, 1.0, seed=seed)
    ro = orc.dsposv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert info == ro.info == 0 and abs(it - ro.iters) <= 1
    assert np.abs(Xg - ro.X).max() / np.abs(ro.X).max() <= 1e-12
    assert certificate(A, Xg, B) < 1.05 and abs(rep.anrm - ro.anrm) <= 1e-13 * ro.anrm


@pytest.mark.parametrize("n,nrhs,seed,variant", [(512, 1, 2, 1), (1000, 3, 3, 1), (2100, 1, 4, 1), (1300, 2, 5, 0),
                                                 (777, 20, 6, 1)])
def test_criterion_spd_wishart(mp, orc, n, nrhs, seed, variant):
    A, B, X = inputs.spd_wishart(n, nrhs=nrhs, seed=seed)
    ro = orc.dsposv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=variant)
    assert info == ro.info == 0
    assert it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters, rep.history(), list(ro.hist))
    assert certificate(A, Xg, B) < 1.05
    h = rep.history()
    assert len(h) == it + 1 and h[-1] < 1.0


@pytest.mark.parametrize("kappa", [1e2, 1e4, 1e6])
def test_criterion_spd_conditioned(mp, orc, kappa):
    n = 1100
    A, B, X = inputs.spd_conditioned(n, kappa, seed=7)
    ro = orc.dsposv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert info == ro.info == 0 and it >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
    assert certificate(A, Xg, B) < 1.05
    bound = kappa * np.linalg.norm(A) * math.sqrt(n) * EPS64           # P8 (||A||_2 = 1)
    assert np.abs(Xg - X).max() / np.abs(X).max() <= bound


def test_spd_8192(mp, orc):
    """C5's size for the SPD form (Wishart stand-in, kappa ~ 34): criterion parity at nb = 256."""
    A, B, X = inputs.spd_wishart(8192, nrhs=1, seed=inputs.BASE_SEED)
    ro = orc.dsposv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert info == ro.info == 0 and abs(it - ro.iters) <= 1, (it, ro.iters)
    assert certificate(A, Xg, B) < 1.05


# ------------------------------------------------------------------------- FALLBACK / errors
def test_fallback_spd(mp, orc):
    n = 600
    A, B, X = inputs.spd_conditioned(n, 1e10, seed=8)
    ro = orc.dsposv(A, B)
    Xg, it, info, rep = gpu_solve(mp, A, B)
    assert it in (-3, -31) and ro.iters in (-3, -31) and info == ro.info == 0
    bound = 1e10 * np.linalg.norm(A) * math.sqrt(n) * EPS64
    assert np.abs(Xg - ro.X).max() / np.abs(ro.X).max() <= bound


def test_forced_fallback_equals_dposv(mp):
    import torch
    A, B, X = inputs.spd_wishart(700, nrhs=2, seed=9)
    Xg, it, info, rep = gpu_solve(mp, A, B, flags=1)
    assert (it, info) == (-31, 0)
    Xd, infod, _ = mp.mp_dposv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    assert infod == 0 and np.array_equal(Xd.cpu().numpy(), Xg)


def test_dposv_vs_oracle(mp, orc):
    import torch
    A, B, X = inputs.spd_wishart(900, nrhs=2, seed=10)
    Xd, info, _ = mp.mp_dposv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    Xo, infoo = orc.dposv(A, B)
    assert info == infoo == 0
    kappa = np.linalg.cond(A)
    assert np.abs(Xd.cpu().numpy() - Xo).max() / np.abs(Xo).max() <= 8 * 900 * kappa * EPS64


def test_only_lower_triangle_read(mp):
    A, B, X = inputs.spd_wishart(450, nrhs=1, seed=11)
    Ag = A.copy(order="F")
    Ag[np.triu_indices(450, 1)] = np.nan
    X1, it1, info1, _ = gpu_solve(mp, A, B)
    X2, it2, info2, _ = gpu_solve(mp, Ag, B)
    assert (it1, info1) == (it2, info2) and np.array_equal(X1, X2)


def test_not_positive_definite(mp, orc):
    A = np.asfortranarray(np.diag([4.0, 1.0, -2.0, 3.0]))
    A[3, 0] = A[0, 3] = 1.0
    b = np.asfortranarray(np.ones((4, 1)))
    Xg, it, info, _ = gpu_solve(mp, A, b)
    ro = orc.dsposv(A, b)
    assert (it, info) == (ro.iters, ro.info) == (-3, 3)
    L, info = mp.mp_spotrf(A)
    assert info == 3


def test_spd_edge_cases(mp):
    Xg, it, info, _ = gpu_solve(mp, np.asfortranarray([[4.0]]), np.asfortranarray([[6.0]]))
    assert (it, info) == (0, 0) and Xg[0, 0] == 1.5
    I = np.asfortranarray(np.eye(129))
    b = np.asfortranarray(np.arange(129, dtype=float)[:, None] / 8)
    Xg, it, info, _ = gpu_solve(mp, I, b)
    assert (it, info) == (0, 0) and np.array_equal(Xg, b)
    A, _, _ = inputs.spd_wishart(200, seed=12)
    Xg, it, info, _ = gpu_solve(mp, A, np.zeros((200, 1), order="F"))
    assert (it, info) == (0, 0) and not Xg.any()
    A2 = A.copy(order="F")
    A2[5, 5] = np.inf
    assert gpu_solve(mp, A2, np.ones((200, 1), order="F"))[2] == -3
