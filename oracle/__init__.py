"""CPU oracle for the mixed-precision iterative-refinement solve (arXiv 0808.2794, Alg. 1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_0808_2794_b200``) never imports it and the
two share no code.  The arithmetic lives in ``oracle/oracle.c`` (plain loops,
fp32 / fp64, see its header for the passages each function follows); this
module only builds that file with gcc and marshals numpy arrays through ctypes.

Layout: matrices are numpy arrays in Fortran (column-major) order, exactly the
C-ABI convention: A is n x n, B and X are n x nrhs with leading dimension n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "oracle_chol.c"), os.path.join(_HERE, "oracle_dd.c"),
         os.path.join(_HERE, "oracle_gmres.c"), os.path.join(_HERE, "oracle_lp.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O3", "-march=x86-64-v2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
           "-fPIC", "-shared", "-std=c11"]
_lock = threading.Lock()
_lib = None

ITERMAX = 30


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i64, p = ctypes.c_int64, ctypes.c_void_p
            pint = ctypes.POINTER(ctypes.c_int)
            lib.oracle_sgetf2.argtypes = [i64, p, i64, p]
            lib.oracle_dgetf2.argtypes = [i64, p, i64, p]
            lib.oracle_sgetrs.argtypes = [i64, i64, p, i64, p, p]
            lib.oracle_dgetrs.argtypes = [i64, i64, p, i64, p, p]
            lib.oracle_residual.argtypes = [i64, i64, p, i64, p, p, p]
            lib.oracle_fro_norm.argtypes = [i64, p, i64]
            lib.oracle_fro_norm.restype = ctypes.c_double
            lib.oracle_dgesv.argtypes = [i64, i64, p, i64, p, p, pint]
            lib.oracle_dsgesv_ex.argtypes = [i64, i64, p, i64, p, p, pint, pint, ctypes.c_int,
                                             p, pint, ctypes.POINTER(ctypes.c_double)]
            lib.oracle_spotf2.argtypes = [i64, p, i64]
            lib.oracle_dpotf2.argtypes = [i64, p, i64]
            lib.oracle_spotrs.argtypes = [i64, i64, p, i64, p]
            lib.oracle_dpotrs.argtypes = [i64, i64, p, i64, p]
            lib.oracle_symv_residual.argtypes = [i64, i64, p, i64, p, p, p]
            lib.oracle_sym_fro_norm.argtypes = [i64, p, i64]
            lib.oracle_sym_fro_norm.restype = ctypes.c_double
            lib.oracle_dposv.argtypes = [i64, i64, p, i64, p, p, pint]
            lib.oracle_dsposv_ex.argtypes = [i64, i64, p, i64, p, p, pint, pint, ctypes.c_int,
                                             p, pint, ctypes.POINTER(ctypes.c_double)]
            pd = ctypes.POINTER(ctypes.c_double)
            d = ctypes.c_double
            lib.oracle_dd_two_sum.argtypes = [d, d, pd, pd]
            lib.oracle_dd_two_prod.argtypes = [d, d, pd, pd]
            lib.oracle_dd_add.argtypes = [d, d, d, d, pd, pd]
            lib.oracle_dd_residual.argtypes = [i64, i64, p, i64, p, p, p, p, p]
            lib.oracle_qdgesv_ex.argtypes = [i64, i64, p, i64, p, p, p, pint, pint, ctypes.c_int, p, pint]
            lib.oracle_gmres_sp_cycle.argtypes = [i64, p, i64, p, ctypes.c_int, p]
            lib.oracle_gmres_sp_cycle.restype = ctypes.c_int
            lib.oracle_fgmres_ex.argtypes = [i64, p, i64, p, p, ctypes.c_int, ctypes.c_int, pint, pint, ctypes.c_int,
                                             p, pint]
            lib.oracle_rna_tf32.argtypes = [ctypes.c_float]
            lib.oracle_rna_tf32.restype = ctypes.c_float
            lib.oracle_rna_tf32_array.argtypes = [i64, p, p]
            lib.oracle_sgetrf_tf32.argtypes = [i64, p, i64, i64, p]
            lib.oracle_sgetrf_tf32.restype = ctypes.c_int
            lib.oracle_dsgesv_tf32_ex.argtypes = [i64, i64, p, i64, p, p, i64, pint, pint, ctypes.c_int, p, pint]
            lib.oracle_gmres_ir_ex.argtypes = [i64, i64, p, i64, p, p, ctypes.c_int, i64, ctypes.c_int, ctypes.c_int,
                                               pint, pint, p, pint]
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _fortran(a, dtype):
    return np.asfortranarray(np.asarray(a, dtype=dtype))


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(t: int) -> None:
    _load().oracle_set_num_threads(int(t))


def sgetf2(A):
    """Step 1 in binary32: returns (LU packed, ipiv 0-based, zero_pivot_info)."""
    LU = _fortran(A, np.float32).copy(order="F")
    n = LU.shape[0]
    ipiv = np.zeros(n, dtype=np.int32)
    info = _load().oracle_sgetf2(n, _ptr(LU), max(1, n), _ptr(ipiv))
    return LU, ipiv, int(info)


def dgetf2(A):
    LU = _fortran(A, np.float64).copy(order="F")
    n = LU.shape[0]
    ipiv = np.zeros(n, dtype=np.int32)
    info = _load().oracle_dgetf2(n, _ptr(LU), max(1, n), _ptr(ipiv))
    return LU, ipiv, int(info)


def sgetrs(LU, ipiv, B):
    LU = _fortran(LU, np.float32)
    n = LU.shape[0]
    Bm = _fortran(B, np.float32).reshape(n, -1, order="F").copy(order="F")
    _load().oracle_sgetrs(n, Bm.shape[1], _ptr(LU), max(1, n), _ptr(np.ascontiguousarray(ipiv, np.int32)), _ptr(Bm))
    return Bm.reshape(np.shape(B), order="F")


def dgetrs(LU, ipiv, B):
    LU = _fortran(LU, np.float64)
    n = LU.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F").copy(order="F")
    _load().oracle_dgetrs(n, Bm.shape[1], _ptr(LU), max(1, n), _ptr(np.ascontiguousarray(ipiv, np.int32)), _ptr(Bm))
    return Bm.reshape(np.shape(B), order="F")


def residual(A, X, B):
    """Step 4: R = B - A X in binary64 with the original A."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Xm = _fortran(X, np.float64).reshape(n, -1, order="F")
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F")
    R = np.empty_like(Bm, order="F")
    _load().oracle_residual(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(Xm), _ptr(R))
    return R.reshape(np.shape(B), order="F")


def fro_norm(A) -> float:
    A = _fortran(A, np.float64)
    return float(_load().oracle_fro_norm(A.shape[0], _ptr(A), max(1, A.shape[0])))


def dgesv(A, B):
    """Full binary64 GEPP solve (the fallback / mp_dgesv semantics). Returns (X, info)."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F")
    X = np.zeros_like(Bm, order="F")
    info = ctypes.c_int(0)
    _load().oracle_dgesv(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(X), ctypes.byref(info))
    return X.reshape(np.shape(B), order="F"), info.value


class Result:
    __slots__ = ("X", "iters", "info", "hist", "anrm")

    def __init__(self, X, iters, info, hist, anrm):
        self.X, self.iters, self.info, self.hist, self.anrm = X, iters, info, hist, anrm

    def __iter__(self):  # allow  X, iters, info = dsgesv(...)
        return iter((self.X, self.iters, self.info))


def dsgesv(A, B, itermax: int = ITERMAX, lda: int | None = None) -> Result:
    """Algorithm 1 with B:5's stop test, cap and fallback."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64)
    Bm = Bm.reshape(n, Bm.size // n if n else (Bm.shape[1] if Bm.ndim > 1 else 1), order="F")
    X = np.zeros_like(Bm, order="F")
    iters, info, nh = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    hist = np.zeros(itermax + 1, dtype=np.float64)
    anrm = ctypes.c_double(0.0)
    _load().oracle_dsgesv_ex(n, Bm.shape[1], _ptr(A), lda if lda is not None else max(1, n), _ptr(Bm), _ptr(X),
                             ctypes.byref(iters), ctypes.byref(info), int(itermax), _ptr(hist),
                             ctypes.byref(nh), ctypes.byref(anrm))
    return Result(X.reshape(np.shape(B), order="F"), iters.value, info.value, hist[: nh.value].copy(), anrm.value)


# ---------------------------------------------------------------------------- SPD variant (oracle_chol.c)
# SPOTRF / SPOTRS / DSYMM in place of SGETRF / SGETRS / DGEMM.  Only the LOWER
# triangle of A is read (LAPACK UPLO = 'L').
def spotf2(A):
    """Step 1, SPD case, binary32: returns (L lower (upper part of the input copy untouched), info)."""
    L = _fortran(A, np.float32).copy(order="F")
    info = _load().oracle_spotf2(L.shape[0], _ptr(L), max(1, L.shape[0]))
    return L, int(info)


def dpotf2(A):
    L = _fortran(A, np.float64).copy(order="F")
    info = _load().oracle_dpotf2(L.shape[0], _ptr(L), max(1, L.shape[0]))
    return L, int(info)


def spotrs(L, B):
    L = _fortran(L, np.float32)
    n = L.shape[0]
    Bm = _fortran(B, np.float32).reshape(n, -1, order="F").copy(order="F")
    _load().oracle_spotrs(n, Bm.shape[1], _ptr(L), max(1, n), _ptr(Bm))
    return Bm.reshape(np.shape(B), order="F")


def dpotrs(L, B):
    L = _fortran(L, np.float64)
    n = L.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F").copy(order="F")
    _load().oracle_dpotrs(n, Bm.shape[1], _ptr(L), max(1, n), _ptr(Bm))
    return Bm.reshape(np.shape(B), order="F")


def symv_residual(A, X, B):
    """Step 4, SPD case: R = B - A_sym X in binary64 from the lower triangle of A."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Xm = _fortran(X, np.float64).reshape(n, -1, order="F")
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F")
    R = np.empty_like(Bm, order="F")
    _load().oracle_symv_residual(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(Xm), _ptr(R))
    return R.reshape(np.shape(B), order="F")


def sym_fro_norm(A) -> float:
    A = _fortran(A, np.float64)
    return float(_load().oracle_sym_fro_norm(A.shape[0], _ptr(A), max(1, A.shape[0])))


def dposv(A, B):
    """Binary64 SPD solver (Cholesky + the two solves): (X, info)."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F")
    X = np.zeros_like(Bm, order="F")
    info = ctypes.c_int(0)
    _load().oracle_dposv(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(X), ctypes.byref(info))
    return X.reshape(np.shape(B), order="F"), info.value


def dsposv(A, B, itermax: int = ITERMAX) -> Result:
    """Algorithm 1, SPD form, with B:5's stop test, cap and fallback."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64)
    Bm = Bm.reshape(n, Bm.size // n if n else (Bm.shape[1] if Bm.ndim > 1 else 1), order="F")
    X = np.zeros_like(Bm, order="F")
    iters, info, nh = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    hist = np.zeros(itermax + 1, dtype=np.float64)
    anrm = ctypes.c_double(0.0)
    _load().oracle_dsposv_ex(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(X), ctypes.byref(iters),
                             ctypes.byref(info), int(itermax), _ptr(hist), ctypes.byref(nh), ctypes.byref(anrm))
    return Result(X.reshape(np.shape(B), order="F"), iters.value, info.value, hist[: nh.value].copy(), anrm.value)


# ---------------------------------------------------------------------------- NEXT-4 (oracle_dd.c)
# P:638-697 "Extension to Quadruple Precision" (QDGESV): binary64 LU + double-double residual / update.
def dd_two_sum(a: float, b: float):
    s, e = ctypes.c_double(), ctypes.c_double()
    _load().oracle_dd_two_sum(a, b, ctypes.byref(s), ctypes.byref(e))
    return s.value, e.value


def dd_two_prod(a: float, b: float):
    s, e = ctypes.c_double(), ctypes.c_double()
    _load().oracle_dd_two_prod(a, b, ctypes.byref(s), ctypes.byref(e))
    return s.value, e.value


def dd_add(a, b):
    s, e = ctypes.c_double(), ctypes.c_double()
    _load().oracle_dd_add(a[0], a[1], b[0], b[1], ctypes.byref(s), ctypes.byref(e))
    return s.value, e.value


def dd_residual(A, Xh, Xl, B):
    """R = B - A (Xh + Xl) in double-double: returns (Rh, Rl)."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F")
    Xh = _fortran(Xh, np.float64).reshape(n, -1, order="F")
    Xl = _fortran(Xl, np.float64).reshape(n, -1, order="F")
    Rh, Rl = np.empty_like(Bm, order="F"), np.empty_like(Bm, order="F")
    _load().oracle_dd_residual(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(Xh), _ptr(Xl), _ptr(Rh), _ptr(Rl))
    return Rh, Rl


class DDResult:
    __slots__ = ("Xh", "Xl", "iters", "info", "hist")

    def __init__(self, Xh, Xl, iters, info, hist):
        self.Xh, self.Xl, self.iters, self.info, self.hist = Xh, Xl, iters, info, hist


def qdgesv(A, B, itermax: int = ITERMAX) -> DDResult:
    """QDGESV analog: binary64 GEPP, double-double residual and update, stop test Q-1."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F")
    Xh, Xl = np.zeros_like(Bm, order="F"), np.zeros_like(Bm, order="F")
    iters, info, nh = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    hist = np.zeros(itermax + 1)
    _load().oracle_qdgesv_ex(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(Xh), _ptr(Xl), ctypes.byref(iters),
                             ctypes.byref(info), int(itermax), _ptr(hist), ctypes.byref(nh))
    return DDResult(Xh, Xl, iters.value, info.value, hist[: nh.value].copy())


# ---------------------------------------------------------------------------- NEXT-3 (oracle_gmres.c)
# Algorithm 2: FGMRES(m_out) in binary64 with one GMRES_SP(m_in) cycle (binary32) per step.
def gmres_sp_cycle(A32, v, m_in: int):
    """One GMRES_SP(m_in) cycle for A32 z = v from z = 0, binary32: returns (z, steps)."""
    A32 = _fortran(A32, np.float32)
    n = A32.shape[0]
    v = np.ascontiguousarray(v, dtype=np.float32)
    z = np.zeros(n, dtype=np.float32)
    steps = _load().oracle_gmres_sp_cycle(n, _ptr(A32), max(1, n), _ptr(v), int(m_in), _ptr(z))
    return z, int(steps)


def fgmres(A, b, m_out: int = 10, m_in: int = 20, itermax: int = ITERMAX) -> Result:
    """Algorithm 2 from x0 = 0; Result.iters = outer cycles (-31: none converged in itermax)."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    bb = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(n))
    x = np.zeros(n, dtype=np.float64)
    iters, info, nh = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    hist = np.zeros(itermax + 1)
    _load().oracle_fgmres_ex(n, _ptr(A), max(1, n), _ptr(bb), _ptr(x), int(m_out), int(m_in), ctypes.byref(iters),
                             ctypes.byref(info), int(itermax), _ptr(hist), ctypes.byref(nh))
    return Result(x.reshape(n, 1), iters.value, info.value, hist[: nh.value].copy(), fro_norm(A))


# ---------------------------------------------------------------------------- NEXT-2 (oracle_lp.c)
# The lower-precision (TF32) factorisation and its refinement: readings T-1..T-4 in oracle_lp.c.
def rna_tf32(x):
    """Round binary32 values to TF32 (nearest, ties away from zero), elementwise."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    out = np.empty_like(a)
    _load().oracle_rna_tf32_array(a.size, _ptr(a), _ptr(out))
    return out


def sgetrf_tf32(A, nb: int):
    """T-1: blocked GEPP (panel nb) of fl32(A) with TF32 trailing updates: (LU packed, ipiv 0-based, info)."""
    LU = _fortran(A, np.float32).copy(order="F")
    n = LU.shape[0]
    ipiv = np.zeros(n, dtype=np.int32)
    info = _load().oracle_sgetrf_tf32(n, _ptr(LU), max(1, n), int(nb), _ptr(ipiv))
    return LU, ipiv, int(info)


def dsgesv_tf32(A, B, nb: int, itermax: int = ITERMAX) -> Result:
    """T-2: Algorithm 1 with the T-1 factors."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F").copy(order="F")
    X = np.zeros_like(Bm, order="F")
    iters, info, nh = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    hist = np.zeros(itermax + 1)
    _load().oracle_dsgesv_tf32_ex(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(X), int(nb), ctypes.byref(iters),
                                  ctypes.byref(info), int(itermax), _ptr(hist), ctypes.byref(nh))
    return Result(X, iters.value, info.value, hist[: nh.value].copy(), fro_norm(A))


def gmres_ir(A, B, nb: int = 0, m: int = 20, itermax: int = ITERMAX, tf32: bool = True) -> Result:
    """T-3/T-4: binary32 LU (TF32 updates with panel nb when tf32, else sgetf2), x0, GMRES-IR(m) per column.
    Result.iters = LU applications (max over columns) or -31 / -3 (X then from the binary64 solver)."""
    A = _fortran(A, np.float64)
    n = A.shape[0]
    Bm = _fortran(B, np.float64).reshape(n, -1, order="F").copy(order="F")
    X = np.zeros_like(Bm, order="F")
    iters, info, nh = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    hist = np.zeros(64)
    _load().oracle_gmres_ir_ex(n, Bm.shape[1], _ptr(A), max(1, n), _ptr(Bm), _ptr(X), 1 if tf32 else 0, int(nb),
                               int(m), int(itermax), ctypes.byref(iters), ctypes.byref(info), _ptr(hist),
                               ctypes.byref(nh))
    return Result(X, iters.value, info.value, hist[: nh.value].copy(), fro_norm(A))
