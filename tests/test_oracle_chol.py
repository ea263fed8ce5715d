"""Pins of the SPD oracle (oracle/oracle_chol.c: P:369-371's SPOTRF / SPOTRS /
DSYMM form of Algorithm 1) against things other than itself: constructed exact factors (bitwise),
exact rational arithmetic, LAPACK through numpy/scipy, closed forms and invariants.  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

EPS32 = 2.0 ** -24
EPS64 = 2.0 ** -53


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


# ---------------------------------------------------------------- constructed exact Cholesky (P2 analog)
@pytest.mark.parametrize("n,seed", [(1, 0), (5, 1), (64, 2), (257, 3)])
def test_exact_cholesky_bitwise(orc, n, seed):
    A, B, X, L = inputs.exact_chol(n, nrhs=2, seed=seed)
    Ls, info = orc.spotf2(A)
    assert info == 0
    assert np.array_equal(np.tril(Ls).astype(np.float64), L)
    Ld, info = orc.dpotf2(A)
    assert info == 0 and np.array_equal(np.tril(Ld), L)
    r = orc.dsposv(A, B)
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X, X)
    Xd, info = orc.dposv(A, B)
    assert info == 0 and np.array_equal(Xd, X)


def test_only_lower_triangle_is_read(orc):
    """UPLO = 'L': garbage (NaN) in the strict upper triangle changes nothing."""
    A, B, X = inputs.spd_wishart(90, nrhs=2, seed=4)
    Ag = A.copy(order="F")
    Ag[np.triu_indices(90, 1)] = np.nan
    r1, r2 = orc.dsposv(A, B), orc.dsposv(Ag, B)
    assert (r1.iters, r1.info) == (r2.iters, r2.info) and np.array_equal(r1.X, r2.X)
    assert np.array_equal(orc.symv_residual(A, X, B), orc.symv_residual(Ag, X, B))
    assert orc.sym_fro_norm(Ag) == orc.sym_fro_norm(A)


# ---------------------------------------------------------------- brute force (exact rationals)
def rational_solve(A, b):
    n = len(b)
    M = [[Fraction(int(A[i, j])) for j in range(n)] + [Fraction(int(b[i]))] for i in range(n)]
    for k in range(n):                       # SPD: no pivoting needed, pivots are positive
        for i in range(k + 1, n):
            f = M[i][k] / M[k][k]
            for j in range(k, n + 1):
                M[i][j] -= f * M[k][j]
    x = [Fraction(0)] * n
    for i in reversed(range(n)):
        x[i] = (M[i][n] - sum(M[i][j] * x[j] for j in range(i + 1, n))) / M[i][i]
    return np.array([float(v) for v in x])


@pytest.mark.parametrize("n,seed", [(2, 0), (3, 1), (5, 2), (6, 3)])
def test_brute_force_small_integer_spd(orc, n, seed):
    rng = np.random.default_rng(seed)
    G = rng.integers(-3, 4, size=(n, n)).astype(float)
    A = np.asfortranarray(G @ G.T + n * np.eye(n))
    b = np.asfortranarray(rng.integers(-3, 4, size=(n, 1)).astype(float))
    x = rational_solve(A, b[:, 0])
    kappa = np.linalg.cond(A)
    Xd, info = orc.dposv(A, b)
    assert info == 0 and np.abs(Xd[:, 0] - x).max() <= 4 * n * kappa * EPS64 * np.abs(x).max()
    r = orc.dsposv(A, b)
    assert r.info == 0 and r.iters >= 0
    assert np.abs(r.X[:, 0] - x).max() <= 4 * n * kappa * EPS64 * np.abs(x).max()


def test_two_by_two_closed_form(orc):
    """[[4, 2], [2, 5]] = L L^T with L = [[2, 0], [1, 2]] (closed form); x = [1, -1] -> b = [2, -3]."""
    A = np.asfortranarray([[4.0, 2.0], [2.0, 5.0]])
    L, info = orc.spotf2(A)
    assert info == 0 and np.array_equal(np.tril(L), np.array([[2.0, 0.0], [1.0, 2.0]], np.float32))
    r = orc.dsposv(A, np.asfortranarray([[2.0], [-3.0]]))
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X[:, 0], [1.0, -1.0])


# ---------------------------------------------------------------- LAPACK special cases (numpy / scipy)
def test_dpotf2_matches_lapack(orc):
    A, _, _ = inputs.spd_wishart(300, seed=5)
    L, info = orc.dpotf2(A)
    Lr = np.linalg.cholesky(A)
    assert info == 0
    assert np.abs(np.tril(L) - Lr).max() <= 300 * EPS64 * np.abs(Lr).max() * 8


def test_spotf2_matches_lapack_float32(orc):
    scipy_linalg = pytest.importorskip("scipy.linalg")
    A, _, _ = inputs.spd_wishart(200, seed=6)
    L, info = orc.spotf2(A)
    Lr = scipy_linalg.cholesky(A.astype(np.float32), lower=True)
    assert info == 0
    assert np.abs(np.tril(L) - Lr).max() <= 200 * EPS32 * np.abs(Lr).max() * 8


def test_dposv_matches_numpy_solve(orc):
    A, B, X = inputs.spd_wishart(250, nrhs=3, seed=7)
    Xd, info = orc.dposv(A, B)
    ref = np.linalg.solve(A, B)
    assert info == 0 and np.abs(Xd - ref).max() <= 64 * 250 * np.linalg.cond(A) * EPS64 * np.abs(ref).max()


def test_symv_residual_matches_long_double(orc):
    A, B, _ = inputs.spd_wishart(180, nrhs=2, seed=8)
    X = np.asfortranarray(np.random.default_rng(1).standard_normal((180, 2)))
    R = orc.symv_residual(A, X, B)
    Rl = np.asarray(B, np.longdouble) - np.asarray(A, np.longdouble) @ np.asarray(X, np.longdouble)
    scale = np.abs(A) @ np.abs(X) + np.abs(B)
    assert np.all(np.abs(R - np.asarray(Rl, float)) <= 180 * EPS64 * scale)


# ---------------------------------------------------------------- invariants
def test_factor_backward_error_invariant(orc):
    A, _, _ = inputs.spd_wishart(400, seed=9)
    L, info = orc.spotf2(A)
    L = np.tril(L).astype(np.float64)
    A32 = A.astype(np.float32).astype(np.float64)
    assert info == 0 and np.linalg.norm(A32 - L @ L.T) / np.linalg.norm(A) <= 10 * 400 * EPS32


def test_stop_test_holds_and_history_decreases(orc):
    A, B, _ = inputs.spd_conditioned(300, 1e4, nrhs=1, seed=10)
    r = orc.dsposv(A, B)
    assert r.info == 0 and r.iters >= 1
    R = np.asarray(B, np.longdouble) - np.asarray(A, np.longdouble) @ np.asarray(r.X, np.longdouble)
    cte = np.linalg.norm(A) * EPS64 * np.sqrt(300)
    assert np.linalg.norm(np.asarray(R, float)) < 1.05 * np.linalg.norm(r.X) * cte
    assert all(h1 > h2 for h1, h2 in zip(r.hist[:-1], r.hist[1:])) and r.hist[-1] < 1.0 <= r.hist[-2]


def test_iterations_monotone_in_kappa_and_fallback(orc):
    n = 256
    U = inputs.haar_orthogonal(n, 11)
    its = []
    for kappa in (1e1, 1e3, 1e5):
        A, B, X = inputs.spd_conditioned(n, kappa, seed=11, U=U)
        r = orc.dsposv(A, B)
        assert r.info == 0 and r.iters >= 0
        its.append(r.iters)
    assert its == sorted(its)
    # kappa eps_s > 1: the binary32 Cholesky breaks down or refinement diverges;
    # either way the binary64 Cholesky solves it
    A, B, X = inputs.spd_conditioned(n, 1e10, seed=11, U=U)
    r = orc.dsposv(A, B)
    assert r.iters in (-3, -31) and r.info == 0
    Xd, _ = orc.dposv(A, B)
    assert np.array_equal(r.X, Xd)


def test_not_positive_definite(orc):
    """An indefinite matrix: the binary32 Cholesky breaks down (iters -3, reading C-1) and so does the
    binary64 one, at the first column whose leading minor is not positive definite (info = k, C-2)."""
    A = np.asfortranarray(np.diag([4.0, 1.0, -2.0, 3.0]))
    A[3, 0] = A[0, 3] = 1.0
    b = np.asfortranarray(np.ones((4, 1)))
    r = orc.dsposv(A, b)
    assert (r.iters, r.info) == (-3, 3)
    assert orc.dposv(A, b)[1] == 3
    L, info = orc.spotf2(A)
    assert info == 3


def test_identity_and_zero_rhs(orc):
    I = np.asfortranarray(np.eye(33))
    b = np.asfortranarray(np.arange(33, dtype=float)[:, None] / 8)
    r = orc.dsposv(I, b)
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X, b)
    A, _, _ = inputs.spd_wishart(40, seed=12)
    r = orc.dsposv(A, np.zeros((40, 1), order="F"))
    assert (r.iters, r.info) == (0, 0) and not r.X.any()


def test_overflow_on_demotion(orc):
    A, B, _ = inputs.spd_wishart(20, seed=13)
    A = A.copy(order="F")
    A[0, 0] = 1e40                                    # beyond FLT_MAX, still SPD
    r = orc.dsposv(A, B)
    assert r.iters == -2 and r.info == 0
    Xd, _ = orc.dposv(A, B)
    assert np.array_equal(r.X, Xd)
