"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names the pin class of DESIGN.md "Oracle pins" (= SURVEY.md §8(c)):
P1 exact rational elimination / Cramer, P2 constructed exact LU (bitwise),
P3 worked examples (tests/golden), P4 closed forms, P5 invariants,
P6 LAPACK special cases, P8 forward-error bound, P9 long-double certificate.
All run on CPU (`-m "not gpu"`).
"""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS32 = 2.0 ** -24
EPS64 = 2.0 ** -53


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def F(rows):
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def perm_from_ipiv(ipiv):
    """Final row order of P A from a sequential LAPACK pivot list (0-based)."""
    p = np.arange(len(ipiv))
    for k, q in enumerate(ipiv):
        p[k], p[q] = p[q], p[k]
    return p


def certificate(A, X, B):
    """P9: b - A x accumulated in long double (x86-64 80-bit), independent of the oracle."""
    Al = np.asarray(A, dtype=np.longdouble)
    Xl = np.asarray(X, dtype=np.longdouble).reshape(A.shape[0], -1)
    Bl = np.asarray(B, dtype=np.longdouble).reshape(A.shape[0], -1)
    R = Bl - Al @ Xl
    return np.asarray(R, dtype=np.float64)


def meets_criterion(A, X, B, slack=1.0):
    """B:5 stop test with the certificate residual: ||r|| < ||x|| ||A||_F 2^-53 sqrt(n) (or r == 0)."""
    n = A.shape[0]
    anrm = float(np.sqrt(np.sum(np.asarray(A, dtype=np.longdouble) ** 2)))
    R = certificate(A, X, B)
    Xm = np.asarray(X).reshape(n, -1)
    for c in range(R.shape[1]):
        rn, xn = np.linalg.norm(R[:, c]), np.linalg.norm(Xm[:, c])
        if not (rn == 0.0 or rn < slack * xn * anrm * EPS64 * math.sqrt(n)):
            return False
    return True


# --------------------------------------------------------------------------- P3
def test_p3_spec_lu_example(oracle):
    g = gold("spec_lu_2x2.json")
    LU, ipiv, info = oracle.sgetf2(F(g["A_rows"]))
    assert info == 0
    assert list(ipiv) == g["ipiv"]
    U = np.triu(LU)
    np.testing.assert_allclose(U, np.array(g["U_rows"]), rtol=0, atol=2 * EPS32 * 6)
    assert LU[1, 0] == np.float32(g["L10"])  # 4/6 rounded once to binary32


def test_p3_spec_solve_examples(oracle):
    for case in gold("spec_solve_2x2.json")["cases"]:
        A, b, x = F(case["A_rows"]), F([[v] for v in case["b"]]), np.array(case["x"], float)
        X, info = oracle.dgesv(A, b)
        assert info == 0
        np.testing.assert_allclose(X[:, 0], x, rtol=0, atol=4 * EPS64 * 10)
        r = oracle.dsgesv(A, b)
        assert r.info == 0 and r.iters >= 0
        np.testing.assert_allclose(r.X[:, 0], x, rtol=0, atol=4 * EPS64 * 10)
        LU, ipiv, _ = oracle.sgetf2(A)
        xs = oracle.sgetrs(LU, ipiv, b.astype(np.float32))
        np.testing.assert_allclose(xs[:, 0], x, rtol=0, atol=1e-5)


def test_p3_spec_residual_examples(oracle):
    for case in gold("spec_residual.json")["cases"]:
        A = F(case["A_rows"])
        R = oracle.residual(A, F([[v] for v in case["x"]]), F([[v] for v in case["b"]]))
        assert np.array_equal(R[:, 0], np.array(case["r"], float))


def test_p3_structurally_singular_column(oracle):
    # lu_factor([[0,1],[0,2]]) -> zero pivot at column 0
    _, _, info = oracle.sgetf2(F([[0, 1], [0, 2]]))
    assert info == 1
    _, _, info = oracle.dgetf2(F([[0, 1], [0, 2]]))
    assert info == 1


# --------------------------------------------------------------------------- P1
def exact_solve(A, b):
    """Gaussian elimination over the rationals (brute force, any pivot) -> exact x or None."""
    n = A.shape[0]
    M = [[Fraction(int(A[i, j])) for j in range(n)] + [Fraction(int(b[i, 0]))] for i in range(n)]
    for k in range(n):
        p = next((i for i in range(k, n) if M[i][k] != 0), None)
        if p is None:
            return None
        M[k], M[p] = M[p], M[k]
        for i in range(k + 1, n):
            f = M[i][k] / M[k][k]
            for j in range(k, n + 1):
                M[i][j] -= f * M[k][j]
    x = [Fraction(0)] * n
    for i in range(n - 1, -1, -1):
        s = M[i][n] - sum(M[i][j] * x[j] for j in range(i + 1, n))
        x[i] = s / M[i][i]
    return x


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_p1_exact_rational_elimination(oracle, n):
    checked = 0
    for seed in range(40):
        A, b = inputs.small_integer_system(n, seed)
        xe = exact_solve(A, b)
        if xe is None:
            continue
        xe = np.array([float(v) for v in xe])
        kappa = np.linalg.cond(A)
        tol = 4 * n * EPS64 * kappa * max(1.0, np.abs(xe).max()) * 4
        X, info = oracle.dgesv(A, b)
        assert info == 0
        assert np.abs(X[:, 0] - xe).max() <= tol
        r = oracle.dsgesv(A, b)
        assert r.info == 0
        if r.iters >= 0:
            assert meets_criterion(A, r.X, b)
            assert np.abs(r.X[:, 0] - xe).max() <= max(tol, 1e-9 * kappa)
        checked += 1
    assert checked >= 20


def test_p1_cramer_2x2_3x3(oracle):
    """adjugate/Cramer on sampled integer 2x2 / 3x3 systems with entries in [-3, 3]."""
    rng = np.random.default_rng(515)
    for n in (2, 3):
        for _ in range(1500):
            A = np.asfortranarray(rng.integers(-3, 4, size=(n, n)).astype(float))
            b = rng.integers(-3, 4, size=(n, 1)).astype(float)
            det = round(np.linalg.det(A))
            if det == 0:
                continue
            # Cramer with exact integer determinants
            xs = []
            for j in range(n):
                Aj = A.copy()
                Aj[:, j] = b[:, 0]
                xs.append(round(np.linalg.det(Aj)) / det)
            r = oracle.dsgesv(A, b)
            assert r.info == 0
            np.testing.assert_allclose(r.X[:, 0], xs, rtol=0, atol=1e-10)


# --------------------------------------------------------------------------- P2
@pytest.mark.parametrize("n", [1, 2, 7, 64, 200, 513])
def test_p2_exact_lu_bitwise(oracle, n):
    A, B, X, perm, L, U = inputs.exact_lu(n, nrhs=2, seed=n)
    LU, ipiv, info = oracle.sgetf2(A)
    assert info == 0
    assert np.array_equal(perm_from_ipiv(ipiv), perm)
    assert np.array_equal(np.tril(LU, -1).astype(np.float64), np.tril(L, -1))
    assert np.array_equal(np.triu(LU).astype(np.float64), U)
    r = oracle.dsgesv(A, B)
    assert (r.iters, r.info) == (0, 0)
    assert np.array_equal(r.X, X)
    Xd, info = oracle.dgesv(A, B)
    assert info == 0 and np.array_equal(Xd, X)
    LUd, ipivd, _ = oracle.dgetf2(A)
    assert np.array_equal(perm_from_ipiv(ipivd), perm)


# --------------------------------------------------------------------------- P4
def test_p4_identity_and_zero_rhs(oracle):
    n = 37
    A = np.asfortranarray(np.eye(n))
    B = np.asfortranarray(np.random.default_rng(1).standard_normal((n, 3)))
    r = oracle.dsgesv(A, B)
    # A = I, generic b: x0 = fl32(b) is off by <= eps32|b|; one correction fl32(b - x0)
    # brings the error to <= eps32^2 |b| (b - x0 has 29 significant bits, rounded once)
    assert r.info == 0 and r.iters == 1
    assert np.abs(r.X - B).max() <= 2 * EPS32 ** 2 * np.abs(B).max()
    assert meets_criterion(A, r.X, B)
    # A = I, fp32-representable b: x0 is exact, r == 0 converges at it = 0 (A-3)
    B32 = np.asfortranarray(B.astype(np.float32).astype(np.float64))
    r = oracle.dsgesv(A, B32)
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X, B32)
    Z = np.zeros((n, 2), order="F")
    Ag, _, _ = inputs.gaussian(n, seed=3)
    r = oracle.dsgesv(Ag, Z)
    assert (r.iters, r.info) == (0, 0) and not r.X.any()  # A-3: r == 0 converges at it = 0


def test_p4_powers_of_two_and_permutation(oracle):
    rng = np.random.default_rng(7)
    n = 50
    D = np.asfortranarray(np.diag(2.0 ** rng.integers(-20, 20, size=n)))
    x = rng.integers(-4, 5, size=(n, 1)) / 4.0
    r = oracle.dsgesv(D, np.asfortranarray(D @ x))
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X, x)
    Pm = np.asfortranarray(np.eye(n)[rng.permutation(n)])
    r = oracle.dsgesv(Pm, np.asfortranarray(Pm @ x))
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X, x)


def test_p4_orthogonal_kappa_one(oracle):
    A, B, X = inputs.conditioned(256, 1.0, seed=11)
    r = oracle.dsgesv(A, B)
    assert r.info == 0 and 1 <= r.iters <= 2
    assert meets_criterion(A, r.X, B)


# --------------------------------------------------------------------------- P5
@pytest.mark.parametrize("n", [64, 300])
def test_p5_factor_quality(oracle, n):
    A, B, X = inputs.gaussian(n, seed=n)
    LU, ipiv, info = oracle.sgetf2(A)
    assert info == 0
    L = np.tril(LU, -1).astype(np.float64) + np.eye(n)
    U = np.triu(LU).astype(np.float64)
    PA = A.astype(np.float32).astype(np.float64)[perm_from_ipiv(ipiv), :]
    rel = np.linalg.norm(PA - L @ U) / np.linalg.norm(A)
    assert rel <= 10 * n * EPS32
    assert np.abs(np.tril(LU, -1)).max() <= 1.0
    # the pivot really is a column maximum at every step (first max wins): replay on the factors
    assert np.all(np.abs(np.diag(U)) > 0)


def test_p5_convergence_and_history(oracle):
    A, B, X = inputs.gaussian(512, seed=2794)
    r = oracle.dsgesv(A, B)
    assert r.info == 0 and 1 <= r.iters <= 4           # CAL: 2-3 at n = 512
    assert len(r.hist) == r.iters + 1
    assert r.hist[-1] < 1.0 and np.all(r.hist[:-1] >= 1.0)
    assert np.all(np.diff(r.hist) < 0)                 # ratio drops every step
    assert meets_criterion(A, r.X, B)
    assert abs(r.anrm - np.linalg.norm(A)) <= 1e-13 * r.anrm


def test_p5_iterations_monotone_in_kappa_and_fallback(oracle):
    n = 200                                            # Fig. condition_number size
    its = {}
    for kappa in (1e1, 1e3, 1e5, 1e8, 1e10):
        vals = []
        for seed in range(3):
            A, B, X = inputs.conditioned(n, kappa, seed=seed)
            r = oracle.dsgesv(A, B)
            assert r.info == 0
            if r.iters >= 0:
                assert meets_criterion(A, r.X, B)
            vals.append(r.iters)
        its[kappa] = vals
    means = [np.mean(its[k]) for k in (1e1, 1e3, 1e5)]
    assert means[0] <= means[1] <= means[2]
    # kappa * eps_s > 1: refinement cannot converge -> -31 and fp64 fallback
    assert its[1e10] == [-31, -31, -31]
    # kappa = 1e8 sits on the kappa*eps_s ~ 1 boundary: no convergence or a very slow one
    assert all(v == -31 or v >= 10 for v in its[1e8])


def test_p5_fallback_solution_is_fp64_quality(oracle):
    n = 200
    A, B, X = inputs.conditioned(n, 1e10, seed=5)
    r = oracle.dsgesv(A, B)
    assert (r.iters, r.info) == (-31, 0)
    Xd, info = oracle.dgesv(A, B)
    assert np.array_equal(r.X, Xd)                     # A-11: fallback = fresh fp64 GEPP + solve
    R = certificate(A, r.X, B)
    assert np.linalg.norm(R) <= 10 * n * EPS64 * np.linalg.norm(A, 2) * np.linalg.norm(r.X)


def test_p5_itermax_cap(oracle):
    A, B, X = inputs.conditioned(200, 1e6, seed=1)
    full = oracle.dsgesv(A, B)
    assert full.iters >= 2
    capped = oracle.dsgesv(A, B, itermax=full.iters - 1)
    assert capped.iters == -31 and capped.info == 0
    exact = oracle.dsgesv(A, B, itermax=full.iters)
    assert exact.iters == full.iters and np.array_equal(exact.X, full.X)


# --------------------------------------------------------------------------- P6
def test_p6_fp64_path_vs_lapack(oracle):
    for n in (10, 100, 257):
        A, B, X = inputs.gaussian(n, nrhs=3, seed=n + 1)
        Xo, info = oracle.dgesv(A, B)
        Xl = np.linalg.solve(A, B)                      # LAPACK dgesv
        kappa = np.linalg.cond(A)
        assert info == 0
        assert np.abs(Xo - Xl).max() / np.abs(Xl).max() <= 8 * n * EPS64 * kappa


def test_p6_fp32_pivots_vs_lapack(oracle):
    scipy_linalg = pytest.importorskip("scipy.linalg")
    for n in (50, 200):
        A, _, _ = inputs.gaussian(n, seed=n + 7)
        A32 = np.asfortranarray(A.astype(np.float32))
        _, ipiv_l = scipy_linalg.lu_factor(A32)         # LAPACK sgetrf (blocked)
        LU, ipiv_o, info = oracle.sgetf2(A)
        assert info == 0
        diff = np.nonzero(ipiv_l != ipiv_o)[0]
        if diff.size:                                   # only near-ties may differ
            k = diff[0]
            col = np.abs(LU[k:, k])
            assert abs(col.max() - np.sort(col)[-2]) <= 1e-4 * col.max()


def test_p6_factor_matches_lapack_on_exact_family(oracle):
    scipy_linalg = pytest.importorskip("scipy.linalg")
    A, B, X, perm, L, U = inputs.exact_lu(128, seed=3)
    lu_l, ipiv_l = scipy_linalg.lu_factor(np.asfortranarray(A.astype(np.float32)))
    LU, ipiv_o, _ = oracle.sgetf2(A)
    assert np.array_equal(ipiv_l, ipiv_o) and np.array_equal(lu_l, LU)


# --------------------------------------------------------------------------- P8
@pytest.mark.parametrize("kappa", [1.0, 10.0, 1e2, 1e4])
def test_p8_forward_error_bound(oracle, kappa):
    n = 256
    A, B, X = inputs.conditioned(n, kappa, seed=2)
    r = oracle.dsgesv(A, B)
    assert r.info == 0 and r.iters >= 0
    fro_over_2 = np.linalg.norm(A) / 1.0                # ||A||_2 = 1 by construction
    bound = kappa * fro_over_2 * math.sqrt(n) * EPS64
    err = np.abs(r.X - X).max() / np.abs(X).max()
    assert err <= bound + 4 * kappa * EPS64             # A-15: b itself is rounded once


# --------------------------------------------------------------------------- errors / edge cases
def test_demotion_overflow_falls_back(oracle):
    A, B, X = inputs.gaussian(20, seed=4)
    A = A.copy(order="F")
    A[3, 5] = 1e39                                      # finite in fp64, inf in fp32
    B = np.asfortranarray(A @ X)
    r = oracle.dsgesv(A, B)
    assert (r.iters, r.info) == (-2, 0)
    Xd, _ = oracle.dgesv(A, B)
    assert np.array_equal(r.X, Xd)


def test_fp32_zero_pivot_falls_back(oracle):
    A = F([[1.0, 1.0], [1.0, 1.0 + 1e-10]])             # singular once demoted
    b = F([[2.0], [2.0 + 1e-10]])
    r = oracle.dsgesv(A, b)
    assert (r.iters, r.info) == (-3, 0)
    np.testing.assert_allclose(r.X[:, 0], [1.0, 1.0], rtol=1e-5)


def test_exactly_singular_reports_info(oracle):
    A = F([[1.0, 2.0], [2.0, 4.0]])
    r = oracle.dsgesv(A, F([[1.0], [2.0]]))
    assert r.iters == -3 and r.info == 2
    _, info = oracle.dgesv(A, F([[1.0], [2.0]]))
    assert info == 2


def test_nonfinite_arguments(oracle):
    A, B, X = inputs.gaussian(8, seed=1)
    A2 = A.copy(order="F"); A2[1, 1] = np.nan
    assert oracle.dsgesv(A2, B).info == -3
    B2 = B.copy(order="F"); B2[0, 0] = np.inf
    assert oracle.dsgesv(A, B2).info == -5


def test_quick_returns(oracle):
    r = oracle.dsgesv(np.zeros((0, 0), order="F"), np.zeros((0, 1), order="F"))
    assert (r.iters, r.info) == (0, 0)
    A, B, X = inputs.gaussian(5, seed=1)
    r = oracle.dsgesv(A, np.zeros((5, 0), order="F"))
    assert (r.iters, r.info) == (0, 0)


def test_thread_count_independence(oracle):
    A, B, X = inputs.gaussian(600, nrhs=2, seed=9)
    t0 = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        r1 = oracle.dsgesv(A, B)
        oracle.set_num_threads(max(2, t0))
        r8 = oracle.dsgesv(A, B)
    finally:
        oracle.set_num_threads(t0)
    assert r1.iters == r8.iters and np.array_equal(r1.X, r8.X)


def test_datta_formula_golden():
    """A-13 reading of P:627-631, recomputed from the printed formula."""
    g = gold("datta.json")
    es, ed = g["eps_s"], g["eps_d"]
    for kappa, it in zip(g["kappa"], g["iterations"]):
        assert math.ceil(math.log(ed) / (math.log(es) + math.log(kappa))) == it
    assert math.log(es) + math.log(g["divergent_from_kappa"]) > 0
    assert math.ceil(math.log(ed) / (math.log(ed) + math.log(10.0))) == g["double_double_kappa10"]
