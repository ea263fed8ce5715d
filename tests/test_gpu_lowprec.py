"""Parity of the lower-precision tensor-core factorisation and its refinement (SURVEY §8(f) NEXT-2:
MP_VARIANT_TF32, 1xTF32 tcgen05 Schur updates; opts.flags bit 8, GMRES-IR; readings T-1..T-4) through the
C-ABI against the oracle (oracle/oracle_lp.c), `-m gpu`.

Bitwise where the result is unique (the P2 exact family: TF32-representable operands make every update
exact), the backward error of the factors against the oracle's TF32 factorisation (same reading, different
accumulation order inside the MMA), B:5's criterion by a long-double certificate, and the correction / LU
application counts against the oracle's within a tolerance stated per test."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

pytestmark = pytest.mark.gpu

EPS64 = 2.0 ** -53
GIR = 256                                  # opts.flags bit 8


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


def default_nb(n):
    return 64 if n <= 1024 else (128 if n <= 4096 else 256)


def perm_from_ipiv(ipiv):
    p = np.arange(len(ipiv))
    for k, q in enumerate(ipiv):
        p[k], p[q] = p[q], p[k]
    return p


def certificate_ok(A, X, B):
    n = A.shape[0]
    Al = np.asarray(A, dtype=np.longdouble)
    R = np.asarray(np.asarray(B, np.longdouble).reshape(n, -1) - Al @ np.asarray(X, np.longdouble).reshape(n, -1),
                   np.float64)
    cte = float(np.sqrt(np.sum(Al * Al))) * EPS64 * math.sqrt(n)
    Xm = np.asarray(X).reshape(n, -1)
    return all(np.linalg.norm(R[:, c]) == 0.0 or np.linalg.norm(R[:, c]) < 1.05 * np.linalg.norm(Xm[:, c]) * cte
               for c in range(R.shape[1]))


def gpu_solve(mp, A, B, **kw):
    import torch
    X, it, info, rep = mp.mp_dsgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B), opts=mp.make_opts(**kw))
    torch.cuda.synchronize()
    return X.cpu().numpy().copy(order="F"), it, info, rep


def backward_error(A, LU, ipiv):
    n = A.shape[0]
    L = np.tril(LU.astype(np.float64), -1) + np.eye(n)
    U = np.triu(LU.astype(np.float64))
    PA = np.asarray(A)[perm_from_ipiv(ipiv)]
    return np.linalg.norm(PA - L @ U) / np.linalg.norm(A)


@pytest.mark.parametrize("n", [700, 2100, 4608])
def test_tf32_exact_family_bitwise(mp, n):
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=1, seed=n + 11)
    LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(variant=mp.MP_VARIANT_TF32))
    assert info == 0
    assert np.array_equal(perm_from_ipiv(ipiv), perm)
    assert np.array_equal(np.tril(LU, -1).astype(np.float64), np.tril(L, -1))
    assert np.array_equal(np.triu(LU).astype(np.float64), U)
    Xg, it, info, _ = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_TF32)
    assert (it, info) == (0, 0) and np.array_equal(Xg, X)


@pytest.mark.parametrize("n,seed", [(1500, 1), (2600, 2)])
def test_tf32_factor_backward_error_matches_oracle(mp, orc, n, seed):
    """Both sides round the update operands to TF32 (T-1): the backward errors agree within 2x, and both are
    far above the 3xTF32 (binary32-accurate) factorisation's."""
    A, _, _ = inputs.gaussian(n, seed=seed)
    LU, ipiv, info = mp.mp_sgetrf(A, mp.make_opts(variant=mp.MP_VARIANT_TF32))
    assert info == 0
    e_gpu = backward_error(A, LU, ipiv)
    LUo, ipo, _ = orc.sgetrf_tf32(A, nb=default_nb(n))
    e_or = backward_error(A, LUo, ipo)
    assert 0.5 * e_or <= e_gpu <= 2.0 * e_or, (e_gpu, e_or)
    LU3, ip3, _ = mp.mp_sgetrf(A, mp.make_opts(variant=mp.MP_VARIANT_3XTF32))
    assert e_gpu > 8 * backward_error(A, LU3, ip3)


@pytest.mark.parametrize("n,shift,seed", [(1200, 3.0, 3), (3000, 2.5, 4)])
def test_tf32_algorithm1_parity(mp, orc, n, shift, seed):
    """T-2: Algorithm 1 with TF32 factors on well-conditioned systems (kappa 2^-11 << 1)."""
    A, B, X = inputs.shifted_gaussian(n, shift=shift, seed=seed)
    ro = orc.dsgesv_tf32(A, B, nb=default_nb(n))
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_TF32)
    assert info == ro.info == 0 and it > 0 and ro.iters > 0
    assert abs(it - ro.iters) <= 2, (it, ro.iters, rep.history(), list(ro.hist))
    assert certificate_ok(A, Xg, B)


@pytest.mark.parametrize("n,kappa,seed,nrhs", [(1200, 1e3, 5, 1), (1500, 3e3, 6, 1), (900, 1e3, 7, 3)])
def test_gmres_ir_parity(mp, orc, n, kappa, seed, nrhs):
    A, B, X = inputs.conditioned(n, kappa, nrhs=nrhs, seed=seed)
    ro = orc.gmres_ir(A, B, nb=default_nb(n), m=20)
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_TF32, flags=GIR)
    assert info == ro.info == 0 and it > 0 and ro.iters > 0
    assert abs(it - ro.iters) <= max(2, ro.iters // 4), (it, ro.iters, rep.history(), list(ro.hist))
    assert certificate_ok(A, Xg, B)


def test_gmres_ir_rescues_large_kappa(mp, orc):
    """kappa 2^-11 ~ 5: Algorithm 1 with the TF32 factors falls back; GMRES-IR(20) converges (cap 63; the
    oracle needs 24 LU applications on this system).  At kappa 2^-11 ~ 25 restarted GMRES(20) stagnates
    too (oracle and GPU): the rescue has a range, not a guarantee."""
    A, B, X = inputs.conditioned(1000, 1e4, seed=8)
    _, it1, info1, _ = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_TF32)
    assert it1 == -31 and info1 == 0
    Xg, it, info, rep = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_TF32, flags=GIR, itermax=63)
    assert info == 0 and 0 < it <= 63, (it, rep.history())
    assert certificate_ok(A, Xg, B)


def test_gmres_ir_with_binary32_factors(mp, orc):
    """GMRES-IR is independent of the factorisation variant: with the 3xTF32 factors it needs no more LU
    applications than Algorithm 1 needs corrections (+1)."""
    A, B, X = inputs.gaussian(2000, seed=9)
    _, it1, _, _ = gpu_solve(mp, A, B)
    Xg, it, info, _ = gpu_solve(mp, A, B, flags=GIR)
    assert info == 0 and 0 < it <= it1 + 1 and certificate_ok(A, Xg, B)
    ro = orc.gmres_ir(A, B, m=20, tf32=False)
    assert abs(it - ro.iters) <= 1


def test_gmres_ir_exact_family_converges_at_x0(mp):
    A, B, X, *_ = inputs.exact_lu(800, nrhs=2, seed=12)
    Xg, it, info, _ = gpu_solve(mp, A, B, variant=mp.MP_VARIANT_TF32, flags=GIR)
    assert (it, info) == (0, 0) and np.array_equal(Xg, X)


def test_tf32_fullsize_well_conditioned(mp):
    """C3's size with TF32 factors on a shifted Gaussian (kappa ~ 2): criterion by the long-double
    certificate on column chunks; corrections within the Datta estimate ceil(ln eps_d / ln(kappa u_f))."""
    import torch
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(inputs.BASE_SEED + 21)
    dA = (torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g) / math.sqrt(n)).t()
    dA.diagonal().add_(3.0)
    x = (torch.rand((1, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    dB = (dA @ x).t().contiguous().t()
    X, it, info, rep = mp.mp_dsgesv_ex(dA, dB, opts=mp.make_opts(variant=mp.MP_VARIANT_TF32))
    torch.cuda.synchronize()
    assert info == 0 and 0 < it <= 10, (it, rep.history())
    A = dA.cpu().numpy()
    B = dB.cpu().numpy()
    Xh = X.cpu().numpy()
    R = np.asarray(B[:, 0], np.longdouble).copy()
    for j0 in range(0, n, 1024):
        R -= np.asarray(A[:, j0:j0 + 1024], np.longdouble) @ np.asarray(Xh[j0:j0 + 1024, 0], np.longdouble)
    cte = np.linalg.norm(A) * EPS64 * math.sqrt(n)
    assert np.linalg.norm(np.asarray(R, np.float64)) < 1.05 * np.linalg.norm(Xh) * cte
