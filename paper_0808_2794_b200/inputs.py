"""Seeded synthetic inputs shared by the GPU path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no LU, no triangular solve,
no residual, no stopping test): it only draws the seeded matrices and vectors
that BASELINE.json's configs describe (B:7-B:11) and forms b = A @ x_true,
which is input generation.  Both sides receive the same bytes.

Layout: A is returned as a Fortran-ordered (column-major) float64 numpy array
of shape (n, n); B / X_true are Fortran-ordered (n, nrhs) float64 arrays — the
C-ABI layout of include/mp_solve.h.

Seeds: base seed s = 2794; A uses s, x_true s+1,
the orthogonal factors of the conditioning sweep s+2 / s+3.  numpy PCG64.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 2794


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _xtrue(n: int, nrhs: int, seed: int) -> np.ndarray:
    return np.asfortranarray(_rng(seed + 1).uniform(-1.0, 1.0, size=(nrhs, n)).T)


def gaussian(n: int, nrhs: int = 1, seed: int = BASE_SEED):
    """C1-C4: A i.i.d. N(0,1) FP64, x_true i.i.d. U[-1,1], b = A x_true (B:7-B:10)."""
    # draw row-major (n, n) and reinterpret its buffer as column-major: A[i, j] = G[j, i]
    G = _rng(seed).standard_normal(size=(n, n))
    A = G.T  # Fortran-ordered view, no copy
    X = _xtrue(n, nrhs, seed)
    B = np.asfortranarray(A @ X)
    return A, B, X


def haar_orthogonal(n: int, seed: int) -> np.ndarray:
    """Q factor of the Householder QR of an N(0,1) matrix, sign-fixed by sign(diag R)."""
    M = _rng(seed).standard_normal(size=(n, n))
    Q, R = np.linalg.qr(M)
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return Q * d[None, :]


def singular_values(n: int, kappa: float) -> np.ndarray:
    """sigma_i = kappa^(-i/(n-1)), i = 0..n-1: geometric from 1 to 1/kappa (B:11)."""
    if n == 1:
        return np.ones(1)
    return kappa ** (-np.arange(n, dtype=np.float64) / (n - 1))


def conditioned(n: int, kappa: float, nrhs: int = 1, seed: int = BASE_SEED, UV=None):
    """C5: A = U diag(sigma) V^T with U, V Haar-orthogonal; ||A||_2 = 1, kappa_2(A) = kappa.

    One (U, V) pair per seed, shared across kappa; pass UV=(U, V) to reuse it.
    """
    if UV is None:
        UV = (haar_orthogonal(n, seed + 2), haar_orthogonal(n, seed + 3))
    U, V = UV
    s = singular_values(n, kappa)
    A = np.asfortranarray((U * s[None, :]) @ V.T)
    X = _xtrue(n, nrhs, seed)
    B = np.asfortranarray(A @ X)
    return A, B, X


def exact_lu(n: int, nrhs: int = 1, seed: int = BASE_SEED, density: float = 0.5):
    """P2 family: A = P^T L U built from short dyadic rationals so every step is exact.

    L: unit lower, off-diagonal entries in {0, +-1/4, +-1/2} (|l| < 1 => the
       partial-pivoting choice is unique and equals P);
    U: integers in [-8, 8], diagonal in {+-1, +-2, +-4};
    P: random permutation; x_true: multiples of 1/4 in [-1, 1].
    Returns (A, B, X, perm, L, U) with A = L U permuted: A[perm[t], :] = (L U)[t, :].
    """
    r = _rng(seed)
    choices_l = np.array([0.25, -0.25, 0.5, -0.5])
    L = np.tril(r.choice(choices_l, size=(n, n)) * (r.random((n, n)) < density), -1) + np.eye(n)
    U = np.triu(r.integers(-8, 9, size=(n, n)).astype(np.float64), 1)
    d = r.choice(np.array([1.0, -1.0, 2.0, -2.0, 4.0, -4.0]), size=n)
    U += np.diag(d)
    perm = r.permutation(n)
    LU = L @ U  # exact: products/sums of short dyadics far below 2^53
    A = np.empty((n, n), order="F")
    A[perm, :] = LU
    X = np.asfortranarray(r.integers(-4, 5, size=(n, nrhs)).astype(np.float64) / 4.0)
    B = np.asfortranarray(A @ X)
    return A, B, X, perm, L, U


def small_integer_system(n: int, seed: int, lo: int = -3, hi: int = 3):
    """P1: integer matrix / rhs with entries in [lo, hi] (exact rational ground truth available)."""
    r = _rng(seed)
    A = np.asfortranarray(r.integers(lo, hi + 1, size=(n, n)).astype(np.float64))
    b = np.asfortranarray(r.integers(lo, hi + 1, size=(n, 1)).astype(np.float64))
    return A, b


def exact_lu_device(n: int, nrhs: int = 1, seed: int = BASE_SEED, density: float = 0.5, device="cuda"):
    """P2 family drawn on the GPU (torch generator) for the full-size configs (C3 16384, C4 49152),
    where the host construction would take minutes.  Same recipe as ``exact_lu``; different bytes.

    L U is formed in binary32 with TF32 disabled: every entry of L is in {0, +-1/4, +-1/2} and U is
    integer in [-8, 8], so every partial sum is a multiple of 1/4 far below 2^22 and the product is
    exact in any summation order.  Returns torch CUDA tensors
    (A column-major float64 (n, n) stride (1, n), B, X (n, nrhs) stride (1, n), perm int64, L, U float32
    row-major) with A[perm[t], :] = (L U)[t, :].
    """
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    s = torch.randint(0, 4, (n, n), device=device, generator=g, dtype=torch.uint8).to(torch.float32)
    L = (s >= 2).to(torch.float32).add_(1.0).mul_(0.25)          # |l| in {1/4, 1/2}
    L.mul_(torch.remainder(s, 2).mul_(-2.0).add_(1.0))           # random sign
    del s
    L.mul_(torch.rand((n, n), device=device, generator=g) < density)
    L.tril_(-1)
    L.diagonal().fill_(1.0)
    U = torch.randint(-8, 9, (n, n), device=device, generator=g, dtype=torch.int8).to(torch.float32)
    U.triu_(1)
    vals_d = torch.tensor([1.0, -1.0, 2.0, -2.0, 4.0, -4.0], device=device)
    U.diagonal().copy_(vals_d[torch.randint(0, 6, (n,), device=device, generator=g)])
    perm = torch.randperm(n, device=device, generator=g)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        Mt = U.t() @ L.t()                  # (L U)^T, row-major: Mt[j, t] = (L U)[t, j]
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    At = torch.empty((n, n), dtype=torch.float64, device=device)
    At[:, perm] = Mt.to(torch.float64)      # At[j, perm[t]] = (L U)[t, j]  ->  A = At^T column-major
    del Mt
    A = At.t()
    Xt = (torch.randint(-4, 5, (nrhs, n), device=device, generator=g).to(torch.float64) / 4.0)
    X = Xt.t()
    Bt = (Xt @ At)                           # B^T = X^T A^T, exact (dyadic, < 2^53)
    B = Bt.t()
    return A, B, X, perm, L, U


# --------------------------------------------------------------------------- SPD variant (NEXT-1)
def spd_wishart(n: int, nrhs: int = 1, seed: int = BASE_SEED):
    """Dense SPD stand-in (the paper's SPD runs state no matrices): A = G G^T / (2n) with G an
    n x 2n N(0,1) matrix — Marchenko-Pastur spectrum in [(1 - 1/sqrt 2)^2, (1 + 1/sqrt 2)^2], kappa ~ 34.
    Full symmetric A (both triangles), x_true U[-1,1], b = A x_true."""
    G = _rng(seed).standard_normal(size=(n, 2 * n))
    A = np.asfortranarray((G @ G.T) / (2.0 * n))
    A = np.asfortranarray(0.5 * (A + A.T))         # exactly symmetric bytes
    X = _xtrue(n, nrhs, seed)
    B = np.asfortranarray(A @ X)
    return A, B, X


def spd_conditioned(n: int, kappa: float, nrhs: int = 1, seed: int = BASE_SEED, U=None):
    """SPD analog of C5: A = U diag(sigma) U^T, U Haar-orthogonal, sigma_i = kappa^(-i/(n-1))."""
    if U is None:
        U = haar_orthogonal(n, seed + 2)
    s = singular_values(n, kappa)
    A = (U * s[None, :]) @ U.T
    A = np.asfortranarray(0.5 * (A + A.T))
    X = _xtrue(n, nrhs, seed)
    B = np.asfortranarray(A @ X)
    return A, B, X


def exact_chol(n: int, nrhs: int = 1, seed: int = BASE_SEED, density: float = 0.5):
    """Pin family for the SPD path: A = L L^T with L lower, diagonal in {1, 2, 4} and off-diagonal entries
    in {0, +-1/4, +-1/2}.  Every step of a Cholesky factorisation (the square roots of l_jj^2, the
    divisions by powers of two, the updates) is exact, so L is reproduced bitwise; x_true is a multiple of
    1/4 in [-1, 1], so the two triangular solves are exact too.  Returns (A full symmetric, B, X, L)."""
    r = _rng(seed)
    choices = np.array([0.25, -0.25, 0.5, -0.5])
    L = np.tril(r.choice(choices, size=(n, n)) * (r.random((n, n)) < density), -1)
    L += np.diag(r.choice(np.array([1.0, 2.0, 4.0]), size=n))
    A = np.asfortranarray(L @ L.T)
    X = np.asfortranarray(r.integers(-4, 5, size=(n, nrhs)).astype(np.float64) / 4.0)
    B = np.asfortranarray(A @ X)
    return A, B, X, L


# --------------------------------------------------------------------------- NEXT-3 (Alg. 2) operators
def shifted_gaussian(n: int, shift: float = 2.5, nrhs: int = 1, seed: int = BASE_SEED):
    """Stand-in for the paper's sparse application matrices (T2, not in the container):
    A = shift I + G / sqrt(n), G i.i.d. N(0,1) — by the circular law its spectrum fills the disk of radius 1
    around `shift`, so restarted GMRES converges geometrically (~1/shift per step) on a dense nonsymmetric
    operator.  x_true U[-1,1], b = A x_true."""
    G = _rng(seed).standard_normal(size=(n, n))
    A = np.asfortranarray(G.T / np.sqrt(n))
    A[np.diag_indices(n)] += shift
    X = _xtrue(n, nrhs, seed)
    B = np.asfortranarray(A @ X)
    return A, B, X
