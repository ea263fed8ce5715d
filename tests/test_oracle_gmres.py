"""Pins of the Algorithm 2 oracle (oracle/oracle_gmres.c: FGMRES-GMRES_SP,
P:240-279) against properties fixed by the mathematics: the GMRES minimal-residual property over the
Krylov space (checked with an independent binary64 least-squares solve), finite termination, closed
forms, monotone outer residuals and agreement with LAPACK's solution.  CPU only."""
import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

EPS64 = 2.0 ** -53


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def krylov_min_residual(A, v, m):
    """min over z in K_m(A, v) of ||v - A z||_2, in binary64 with an orthonormal Krylov basis (numpy QR)."""
    n = len(v)
    Q = np.zeros((n, m))                       # Arnoldi (MGS, twice) in binary64: an orthonormal K_m basis
    w = v / np.linalg.norm(v)
    for j in range(m):
        Q[:, j] = w
        w = A @ w
        for _ in range(2):
            w = w - Q[:, :j + 1] @ (Q[:, :j + 1].T @ w)
        w = w / np.linalg.norm(w)
    y, *_ = np.linalg.lstsq(A @ Q, v, rcond=None)
    return np.linalg.norm(v - A @ (Q @ y))


@pytest.mark.parametrize("n,m,seed", [(60, 5, 0), (120, 12, 1), (200, 20, 2)])
def test_gmres_sp_cycle_is_minimal_residual(orc, n, m, seed):
    A, _, _ = inputs.shifted_gaussian(n, shift=1.5, seed=seed)
    v = np.random.default_rng(seed).standard_normal(n)
    A32 = A.astype(np.float32)
    z, steps = orc.gmres_sp_cycle(A32, v.astype(np.float32), m)
    assert steps == m
    A32d = A32.astype(np.float64)
    res = np.linalg.norm(v.astype(np.float32).astype(np.float64) - A32d @ z.astype(np.float64))
    best = krylov_min_residual(A32d, v.astype(np.float32).astype(np.float64), m)
    nv = np.linalg.norm(v)
    assert res >= best - 1e-6 * nv                          # nothing beats the minimum (up to binary32 noise) ...
    assert res <= best + 2e-5 * nv                          # ... and the binary32 cycle reaches it


def test_gmres_sp_finite_termination(orc):
    """A with 3 distinct eigenvalues (diagonal): the Krylov space holds the solution after 3 steps, so a
    3-step cycle solves A z = v to binary32 accuracy (exactly-zero h_{4,3}, a happy breakdown, needs exact
    arithmetic; in binary32 it is ~1e-7 and a longer cycle stays accurate)."""
    d = np.array([1.0, 2.0, 4.0] * 10)
    A = np.asfortranarray(np.diag(d))
    v = np.linspace(-1.0, 1.0, 30).astype(np.float32)
    z, steps = orc.gmres_sp_cycle(A.astype(np.float32), v, 3)
    assert steps == 3 and np.allclose(z, v / d, rtol=0, atol=2e-6)
    z2, _ = orc.gmres_sp_cycle(A.astype(np.float32), v, 2)
    assert np.abs(z2 - v / d).max() > 1e-3                 # 2 steps cannot
    z, steps = orc.gmres_sp_cycle(np.asfortranarray(np.eye(30, dtype=np.float32)), v, 5)
    assert np.allclose(z, v, rtol=0, atol=4e-7)           # A = I: one step suffices


@pytest.mark.parametrize("n,m_out,m_in,seed", [(100, 4, 10, 3), (256, 10, 20, 4), (300, 20, 30, 5)])
def test_fgmres_converges_to_the_solution(orc, n, m_out, m_in, seed):
    A, B, X = inputs.shifted_gaussian(n, seed=seed)
    r = orc.fgmres(A, B, m_out=m_out, m_in=m_in)
    assert r.info == 0 and r.iters >= 1
    R = np.asarray(B[:, 0], np.longdouble) - np.asarray(A, np.longdouble) @ np.asarray(r.X[:, 0], np.longdouble)
    cte = np.linalg.norm(A) * EPS64 * np.sqrt(n)
    assert np.linalg.norm(np.asarray(R, float)) < 1.05 * np.linalg.norm(r.X) * cte     # B:5's test (G-1)
    ref = np.linalg.solve(A, B[:, 0])
    assert np.abs(r.X[:, 0] - ref).max() <= 64 * n * np.linalg.cond(A) * EPS64 * np.abs(ref).max()
    h = r.hist
    assert h[-1] < 1.0 and all(a > b for a, b in zip(h[:-1], h[1:]))                   # monotone outer residual


def test_fgmres_closed_forms(orc):
    n = 50
    b = np.linspace(-1, 1, n).reshape(n, 1)
    r = orc.fgmres(np.asfortranarray(np.eye(n)), b, m_out=3, m_in=3)
    assert r.info == 0 and 1 <= r.iters <= 3 and np.abs(r.X - b).max() <= 4 * EPS64
    r = orc.fgmres(np.asfortranarray(np.eye(n) * 4.0), np.zeros((n, 1)), m_out=3, m_in=3)
    assert (r.iters, r.info) == (0, 0) and not r.X.any()


def test_fgmres_cap(orc):
    """A hard operator (eigenvalues around 0) with tiny restarts: no convergence within the cap (G-2)."""
    A, B, _ = inputs.shifted_gaussian(80, shift=0.0, seed=6)
    r = orc.fgmres(A, B, m_out=1, m_in=1, itermax=5)
    assert r.iters == -31 and len(r.hist) == 6
