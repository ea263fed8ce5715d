"""Parity of the extended-precision refinement (the paper's QDGESV, with
quadruple precision as double-double, reading Q-0) through the C-ABI against the oracle (oracle_dd.c)
and against exact rational arithmetic, `-m gpu`."""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

pytestmark = pytest.mark.gpu

U104 = 2.0 ** -104


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


def gpu_qd(mp, A, B, **kw):
    import torch
    Xh, Xl, it, info, rep = mp.mp_qdgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B),
                                            opts=mp.make_opts(**kw) if kw else None)
    torch.cuda.synchronize()
    return Xh.cpu().numpy().copy(order="F"), Xl.cpu().numpy().copy(order="F"), it, info, rep


def dd_certificate(orc, A, Xh, Xl, B):
    """The oracle's double-double residual of the GPU solution against the Q-1 threshold."""
    n = A.shape[0]
    Rh, _ = orc.dd_residual(A, Xh, Xl, B)
    cte = np.linalg.norm(A) * U104 * math.sqrt(n)
    return max(np.linalg.norm(Rh[:, c]) / (np.linalg.norm(Xh[:, c]) * cte) if np.linalg.norm(Rh[:, c]) else 0.0
               for c in range(Rh.shape[1]))


@pytest.mark.parametrize("n,nrhs,seed", [(300, 1, 0), (1000, 3, 1), (2100, 1, 2), (1300, 2, 3)])
def test_qd_parity_gaussian(mp, orc, n, nrhs, seed):
    A, B, X = inputs.gaussian(n, nrhs=nrhs, seed=seed)
    ro = orc.qdgesv(A, B)
    Xh, Xl, it, info, rep = gpu_qd(mp, A, B)
    assert info == ro.info == 0
    assert it >= 0 and ro.iters >= 0 and abs(it - ro.iters) <= 1, (it, ro.iters, rep.history(), list(ro.hist))
    assert dd_certificate(orc, A, Xh, Xl, B) < 1.05
    # the two double-double solutions agree far beyond binary64: (xh_g - xh_o) + (xl_g - xl_o)
    gap = np.abs((Xh - ro.Xh) + (Xl - ro.Xl)).max() / np.abs(ro.Xh).max()
    kappa = np.linalg.cond(A)
    assert gap <= 8 * n * kappa * U104 * math.sqrt(n), gap
    assert gap < 1e-20


def test_qd_against_exact_rationals(mp):
    n = 40
    A, B, _ = inputs.gaussian(n, nrhs=1, seed=5)
    Xh, Xl, it, info, rep = gpu_qd(mp, A, B)
    assert info == 0 and 0 <= it <= 3                                   # "No more than 3 steps"
    F = lambda v: Fraction(float(v))
    M = [[F(A[i, j]) for j in range(n)] + [F(B[i, 0])] for i in range(n)]
    for k in range(n):
        p = max(range(k, n), key=lambda i: abs(M[i][k]))
        M[k], M[p] = M[p], M[k]
        for i in range(k + 1, n):
            f = M[i][k] / M[k][k]
            for j in range(k, n + 1):
                M[i][j] -= f * M[k][j]
    x = [Fraction(0)] * n
    for i in reversed(range(n)):
        x[i] = (M[i][n] - sum(M[i][j] * x[j] for j in range(i + 1, n))) / M[i][i]
    err = max(abs(F(Xh[i, 0]) + F(Xl[i, 0]) - x[i]) for i in range(n)) / max(abs(v) for v in x)
    assert err <= Fraction(8 * n * np.linalg.cond(A) * U104), float(err)


def test_qd_edge_cases(mp, orc):
    import torch
    I = np.asfortranarray(np.eye(100))
    b = np.asfortranarray(np.arange(100, dtype=float)[:, None] / 3)
    Xh, Xl, it, info, _ = gpu_qd(mp, I, b)
    assert (it, info) == (0, 0) and np.array_equal(Xh, b) and not Xl.any()
    S = np.asfortranarray([[1.0, 2.0], [2.0, 4.0]])
    assert gpu_qd(mp, S, np.ones((2, 1), order="F"))[3] == 2
    A, B, _ = inputs.gaussian(200, nrhs=2, seed=6)
    Xh, Xl, it, info, _ = gpu_qd(mp, A, np.zeros((200, 2), order="F"))
    assert (it, info) == (0, 0) and not Xh.any()
    # host buffers: the library stages the copies (same result as device buffers)
    Xh_d, Xl_d, it_d, _, _ = gpu_qd(mp, A, B)
    Xh_h, Xl_h, it_h, info_h, _ = mp.mp_qdgesv_ex(A, B)
    assert (it_h, info_h) == (it_d, 0) and np.array_equal(Xh_h, Xh_d) and np.array_equal(Xl_h, Xl_d)


def test_qd_beats_binary64_accuracy(mp, orc):
    """Against a double-double reference (the oracle), the GPU's x is ~1e-12 / kappa closer than the
    binary64 solve of mp_dgesv: the point of the extension."""
    import torch
    A, B, _ = inputs.gaussian(800, nrhs=1, seed=7)
    ro = orc.qdgesv(A, B)
    Xh, Xl, it, info, _ = gpu_qd(mp, A, B)
    Xd, infod, _ = mp.mp_dgesv_ex(mp.colmajor_cuda(A), mp.colmajor_cuda(B))
    torch.cuda.synchronize()
    Xd = Xd.cpu().numpy()
    err_qd = np.abs((Xh - ro.Xh) + (Xl - ro.Xl)).max()
    err_64 = np.abs((Xd - ro.Xh) - ro.Xl).max()
    assert err_qd * 1e6 < err_64
