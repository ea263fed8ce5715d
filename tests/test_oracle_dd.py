"""Pins of the extended-precision oracle (oracle/oracle_dd.c: the paper's QDGESV,
P:638-697, with quadruple precision carried as double-double, reading Q-0) against exact rational
arithmetic (Python fractions) and closed forms.  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

U104 = 2.0 ** -104


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def F(x):
    return Fraction(float(x))


def test_error_free_transformations(orc):
    rng = np.random.default_rng(0)
    for _ in range(2000):
        a, b = rng.standard_normal() * 10.0 ** rng.integers(-20, 20), rng.standard_normal() * 10.0 ** rng.integers(-20, 20)
        s, e = orc.dd_two_sum(a, b)
        assert F(s) + F(e) == F(a) + F(b) and s == a + b
        p, e = orc.dd_two_prod(a, b)
        assert F(p) + F(e) == F(a) * F(b) and p == a * b


def test_dd_add_accuracy(orc):
    rng = np.random.default_rng(1)
    for _ in range(2000):
        ah = rng.standard_normal(); al = ah * 2.0 ** -60 * rng.standard_normal()
        ah, al = orc.dd_two_sum(ah, al)
        bh = rng.standard_normal() * (1 if rng.random() < 0.5 else -1); bl = bh * 2.0 ** -60 * rng.standard_normal()
        bh, bl = orc.dd_two_sum(bh, bl)
        sh, sl = orc.dd_add((ah, al), (bh, bl))
        exact = F(ah) + F(al) + F(bh) + F(bl)
        got = F(sh) + F(sl)
        assert abs(got - exact) <= 4 * U104 * abs(exact) + Fraction(2) ** -1074
        assert abs(sl) <= abs(sh) * 2.0 ** -52


def exact_residual(A, x, b):
    n = A.shape[0]
    return [F(b[i]) - sum(F(A[i, j]) * x[j] for j in range(n)) for i in range(n)]


def test_dd_residual_matches_exact(orc):
    rng = np.random.default_rng(2)
    n = 24
    A = np.asfortranarray(rng.standard_normal((n, n)))
    b = np.asfortranarray(rng.standard_normal((n, 1)))
    xh = np.asfortranarray(rng.standard_normal((n, 1)))
    xl = np.asfortranarray(xh * 2.0 ** -55 * rng.standard_normal((n, 1)))
    Rh, Rl = orc.dd_residual(A, xh, xl, b)
    x = [F(xh[j, 0]) + F(xl[j, 0]) for j in range(n)]
    r = exact_residual(A, x, b[:, 0])
    scale = np.abs(A) @ np.abs(xh[:, 0]) + np.abs(b[:, 0])
    for i in range(n):
        assert abs(F(Rh[i, 0]) + F(Rl[i, 0]) - r[i]) <= Fraction(4 * n * U104 * scale[i])


def rational_solve(A, b):
    n = len(b)
    M = [[F(A[i, j]) for j in range(n)] + [F(b[i])] for i in range(n)]
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
    return x


@pytest.mark.parametrize("n,seed", [(3, 0), (10, 1), (40, 2)])
def test_qdgesv_against_exact_rationals(orc, n, seed):
    A, B, _ = inputs.gaussian(n, nrhs=1, seed=seed)
    r = orc.qdgesv(A, B)
    assert r.info == 0 and 0 <= r.iters <= 3                       # "No more than 3 steps"
    x = rational_solve(A, B[:, 0])
    kappa = np.linalg.cond(A)
    xmax = max(abs(v) for v in x)
    err = max(abs(F(r.Xh[i, 0]) + F(r.Xl[i, 0]) - x[i]) for i in range(n))
    assert err <= Fraction(8 * n * kappa * U104) * xmax, float(err / xmax)
    # beyond binary64: the double-double solution is far more accurate than the binary64 one
    Xd, _ = orc.dgesv(A, B)
    err64 = max(abs(F(Xd[i, 0]) - x[i]) for i in range(n))
    assert err < err64 or err64 == 0


def test_qdgesv_ill_conditioned_hilbert(orc):
    """Hilbert n = 8 (kappa ~ 1.5e10 < 1/u_d): refinement still converges to double-double accuracy
    (Datta-style count ceil(ln u_dd / ln(kappa u_d)) ~ 7 at most), checked against exact rationals."""
    n = 8
    A = np.asfortranarray([[1.0 / (i + j + 1) for j in range(n)] for i in range(n)])
    b = np.asfortranarray(np.ones((n, 1)))
    r = orc.qdgesv(A, b)
    assert r.info == 0 and 1 <= r.iters <= 10
    x = rational_solve(A, b[:, 0])
    xmax = max(abs(v) for v in x)
    err = max(abs(F(r.Xh[i, 0]) + F(r.Xl[i, 0]) - x[i]) for i in range(n))
    assert err <= Fraction(8 * n * 1.6e10 * U104) * xmax


def test_qdgesv_closed_forms(orc):
    I = np.asfortranarray(np.eye(17))
    b = np.asfortranarray(np.arange(17, dtype=float)[:, None] / 3)
    r = orc.qdgesv(I, b)
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.Xh, b) and not r.Xl.any()
    S = np.asfortranarray([[1.0, 2.0], [2.0, 4.0]])
    assert orc.qdgesv(S, np.ones((2, 1), order="F")).info == 2
    A, _, _ = inputs.gaussian(30, seed=3)
    r = orc.qdgesv(A, np.zeros((30, 2), order="F"))
    assert (r.iters, r.info) == (0, 0) and not r.Xh.any()


def test_qdgesv_stop_test_and_history(orc):
    A, B, _ = inputs.gaussian(120, nrhs=2, seed=4)
    r = orc.qdgesv(A, B)
    assert r.info == 0 and r.iters >= 1
    assert r.hist[-1] < 1.0 and all(h >= 1.0 for h in r.hist[:-1])
    assert all(h1 > h2 for h1, h2 in zip(r.hist[:-1], r.hist[1:]))
