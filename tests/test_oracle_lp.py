"""Pins of the NEXT-2 oracle (oracle/oracle_lp.c: the lower-precision TF32
factorisation and its refinement, readings T-1..T-4) against what arithmetic and mathematics fix:
hand-computed roundings, an independent (frexp-based) derivation of round-to-nearest-away, reduction to
the unblocked binary32 elimination, exact factors of the P2 family, a hand-computed TF32 Schur update,
the backward-error magnitude u_f = 2^-11, the FGMRES(1) closed form and convergence.  CPU only."""
import numpy as np
import pytest

from paper_0808_2794_b200 import inputs

EPS64 = 2.0 ** -53


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def test_rna_tf32_hand_values(orc):
    u = 2.0 ** -10                                        # TF32 ulp at 1
    x = np.array([1 + 2.0 ** -12, 1 + 2.5 * u, -(1 + 2.5 * u), 1 + 0.5 * u, 1 + 0.25 * u, 1 + u, 0.0, -0.0,
                  2.0 ** -130, 3.0], np.float32)
    want = np.array([1.0, 1 + 3 * u, -(1 + 3 * u), 1 + u, 1.0, 1 + u, 0.0, -0.0, 2.0 ** -130, 3.0], np.float32)
    got = orc.rna_tf32(x)
    assert np.array_equal(got, want)
    assert np.signbit(got[7])
    assert np.isinf(orc.rna_tf32([np.inf]))[0] and np.isnan(orc.rna_tf32([np.nan]))[0]


def test_rna_tf32_matches_frexp_derivation(orc):
    """round(x) to 11 significant bits, ties away, derived with frexp/ldexp in binary64."""
    r = np.random.default_rng(3)
    x = (r.standard_normal(20000) * np.exp2(r.integers(-20, 20, 20000))).astype(np.float32)
    x[:50] = (1 + (2 * r.integers(0, 1024, 50) + 1) * 2.0 ** -11).astype(np.float32)   # exact ties
    m, e = np.frexp(x.astype(np.float64))                 # x = m 2^e, 0.5 <= |m| < 1
    q = np.sign(m) * np.floor(np.abs(m) * 2.0 ** 11 + 0.5)
    want = np.ldexp(q, e - 11).astype(np.float32)
    assert np.array_equal(orc.rna_tf32(x), want)


def test_sgetrf_tf32_single_panel_is_sgetf2(orc):
    A, _, _ = inputs.gaussian(70, seed=4)
    LU1, p1, i1 = orc.sgetrf_tf32(A, nb=70)
    LU2, p2, i2 = orc.sgetf2(A)
    assert i1 == i2 == 0 and np.array_equal(p1, p2) and np.array_equal(LU1, LU2)


@pytest.mark.parametrize("n,nb", [(96, 16), (130, 32), (64, 7)])
def test_sgetrf_tf32_exact_family(orc, n, nb):
    """P2 family: L, U and every Schur complement are short dyadics (TF32-representable operands), so the
    TF32 factorisation is exact: the factors are L and U, the pivots P."""
    A, _, _, perm, L, U = inputs.exact_lu(n, seed=n)
    LU, ipiv, info = orc.sgetrf_tf32(A, nb=nb)
    assert info == 0
    assert np.array_equal(np.tril(LU, -1) + np.eye(n), L) and np.array_equal(np.triu(LU), U)
    p = np.arange(n)
    for k in range(n):
        p[[k, ipiv[k]]] = p[[ipiv[k], k]]
    assert np.array_equal(p, perm)


def test_sgetrf_tf32_hand_update(orc):
    """nb = 1, no interchange: U[1,1] = a22 - rna(l) rna(u) with l = 0.5 + 2^-13 -> 0.5 and
    u = 1 + 5 2^-11 -> 1 + 3 2^-10; the stored factors keep the binary32 values."""
    l, u = np.float32(0.5 + 2.0 ** -13), np.float32(1 + 5 * 2.0 ** -11)
    A = np.array([[1.0, u], [l, 3.0]], order="F")
    LU, ipiv, info = orc.sgetrf_tf32(A, nb=1)
    assert info == 0 and list(ipiv) == [0, 1]
    assert LU[1, 0] == l and LU[0, 1] == u
    assert LU[1, 1] == np.float32(2.5 - 1.5 * 2.0 ** -10)
    LU2, _, _ = orc.sgetf2(A)
    assert LU2[1, 1] != LU[1, 1]                         # binary32 elimination differs


def test_sgetrf_tf32_backward_error_scale(orc):
    """||P A - L U||_F / ||A||_F: ~u_f = 2^-11 scale for TF32 updates, far above the binary32 LU's."""
    n = 256
    A, _, _ = inputs.gaussian(n, seed=9)
    def berr(LU, ipiv):
        L = np.tril(LU.astype(np.float64), -1) + np.eye(n)
        U = np.triu(LU.astype(np.float64))
        PA = A.copy()
        for k in range(n):
            PA[[k, ipiv[k]]] = PA[[ipiv[k], k]]
        return np.linalg.norm(PA - L @ U) / np.linalg.norm(A)
    e_tf = berr(*orc.sgetrf_tf32(A, nb=32)[:2])
    e_32 = berr(*orc.sgetf2(A)[:2])
    assert 2.0 ** -16 < e_tf < 2.0 ** -7
    assert e_tf > 16 * e_32


def test_dsgesv_tf32_converges_on_well_conditioned(orc):
    A, B, X = inputs.shifted_gaussian(300, shift=3.0, seed=5)
    r = orc.dsgesv_tf32(A, B, nb=32)
    assert r.info == 0 and 1 <= r.iters <= 12
    assert np.abs(r.X - X).max() <= 1e-12
    r32 = orc.dsgesv(A, B)
    assert r32.iters <= r.iters                          # coarser factors never need fewer corrections here


def test_gmres_ir_moderate_kappa_no_worse_than_ir(orc):
    """kappa 2^-11 ~ 5: both converge; the minimal-residual outer solver needs no more LU applications
    than Algorithm 1 needs corrections (+1 for the restart check)."""
    A, B, _ = inputs.conditioned(300, 1e4, seed=21)
    ir = orc.dsgesv_tf32(A, B, nb=32)
    g = orc.gmres_ir(A, B, nb=32, m=20)
    assert ir.iters > 0 and g.iters > 0 and g.iters <= ir.iters + 1


def test_gmres_ir_exact_factors_converge_at_x0(orc):
    A, B, X, *_ = inputs.exact_lu(80, seed=2)
    r = orc.gmres_ir(A, B, nb=16, m=10)
    assert (r.iters, r.info) == (0, 0) and np.array_equal(r.X, X)


def test_gmres_ir_m1_closed_form(orc):
    """FGMRES(1): each cycle x <- x + y z with z = LUsolve(fl32(r/||r||)) and y = argmin ||r - y A z||
    = (A z)^T r / ||A z||^2.  One capped cycle from x0, recomputed here with numpy and oracle.sgetrs."""
    n = 120
    A, B, _ = inputs.gaussian(n, seed=12)
    LU, ipiv, _ = orc.sgetrf_tf32(A, nb=16)
    x0 = orc.sgetrs(LU, ipiv, B.astype(np.float32)).astype(np.float64)[:, 0]
    r = B[:, 0] - A @ x0
    v = r / np.linalg.norm(r)
    z = orc.sgetrs(LU, ipiv, v.astype(np.float32).reshape(n, 1)).astype(np.float64)[:, 0]
    w = A @ z
    y = (w @ r) / (w @ w)
    # compared through the history: hist[1] = ||b - A x1|| / (||x1|| cte) after the first cycle
    x1 = x0 + y * z
    cte = np.linalg.norm(A) * EPS64 * np.sqrt(n)
    want = np.linalg.norm(B[:, 0] - A @ x1) / (np.linalg.norm(x1) * cte)
    res = orc.gmres_ir(A, B, nb=16, m=1, itermax=30)
    assert res.hist.size >= 2
    assert abs(res.hist[1] - want) <= 1e-6 * want + 1e-3


def test_gmres_ir_beats_ir_when_kappa_uf_large(orc):
    """kappa(A) 2^-11 >> 1: Algorithm 1 with TF32 factors diverges (fallback), GMRES-IR(30) converges
    (with a larger application cap: the preconditioned operator is far from the identity)."""
    n = 300
    A, B, X = inputs.conditioned(n, 1e5, seed=21)
    kappa = np.linalg.cond(A)
    assert kappa * 2.0 ** -11 > 20
    ir = orc.dsgesv_tf32(A, B, nb=32)
    g = orc.gmres_ir(A, B, nb=32, m=30, itermax=63)
    assert g.iters >= 1 and g.info == 0
    assert ir.iters == -31
    R = np.asarray(B[:, 0], np.longdouble) - np.asarray(A, np.longdouble) @ np.asarray(g.X[:, 0], np.longdouble)
    cte = np.linalg.norm(A) * EPS64 * np.sqrt(n)
    assert np.linalg.norm(np.asarray(R, float)) < 1.05 * np.linalg.norm(g.X) * cte
