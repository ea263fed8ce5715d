"""Thin ctypes binding of libmpsolve.so (include/mp_solve.h) — argument marshalling only.

Names mirror the C-ABI.  Matrices are column-major (Fortran order):
* torch CUDA tensors: A of shape (n, n) with stride (1, lda); B, X of shape
  (n, nrhs) with stride (1, n) — see ``colmajor_cuda`` to build them;
* numpy arrays (host): Fortran-ordered float64 — the library stages the
  host<->device copies itself (the end-to-end path).

Every step of the solve runs in the CUDA kernels of libmpsolve.so.  If the
library is missing this module raises at import time: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpsolve.so")

MP_OK, MP_ERR_CUDA, MP_ERR_NOMEM, MP_ERR_INTERNAL, MP_ERR_NCCL, MP_ERR_UNSUPPORTED = 0, 1, 2, 3, 4, 5
MP_VARIANT_FFMA, MP_VARIANT_3XTF32, MP_VARIANT_TF32 = 0, 1, 2
MP_HIST_MAX = 64
KCLASSES = ("demote", "panel", "laswp", "trsm", "gemm", "solve", "residual", "trail")


class Opts(ctypes.Structure):
    _fields_ = [("nb", ctypes.c_int32), ("itermax", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("flags", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("info", ctypes.c_int32), ("nhist", ctypes.c_int32),
                ("nb", ctypes.c_int32), ("variant", ctypes.c_int32), ("solve_inv", ctypes.c_int32),
                ("anrm", ctypes.c_double), ("hist", ctypes.c_double * MP_HIST_MAX),
                ("t_total_ms", ctypes.c_double), ("t_demote_ms", ctypes.c_double),
                ("t_factor_ms", ctypes.c_double), ("t_refine_ms", ctypes.c_double),
                ("t_fallback_ms", ctypes.c_double), ("t_copy_ms", ctypes.c_double),
                ("workspace_bytes", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("k_ms", ctypes.c_double * 8), ("k_work", ctypes.c_double * 8), ("k_launches", ctypes.c_int64 * 8)]

    def history(self):
        return [self.hist[i] for i in range(self.nhist)]

    def kernels(self):
        return {KCLASSES[i]: {"ms": self.k_ms[i], "work": self.k_work[i], "launches": self.k_launches[i]}
                for i in range(8) if self.k_launches[i]}


class MpError(RuntimeError):
    pass


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_0808_2794_b200.build` "
                      "(there is no CPU fallback for the CUDA path)")

lib = ctypes.CDLL(LIB_PATH)
_i64, _p, _pi = ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)
lib.mp_default_opts.argtypes = [ctypes.POINTER(Opts)]
lib.mp_default_opts.restype = None
lib.mp_dsgesv.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi, _pi]
lib.mp_dsgesv_ex.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi, _pi, ctypes.POINTER(Opts), ctypes.POINTER(Report)]
lib.mp_dgesv.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi]
lib.mp_dgesv_ex.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi, ctypes.POINTER(Opts), ctypes.POINTER(Report)]
lib.mp_sgetrf.argtypes = [_i64, _p, _i64, _p, _p, _pi, ctypes.POINTER(Opts)]
lib.mp_dgetrf.argtypes = [_i64, _p, _i64, _p, _p, _pi, ctypes.POINTER(Opts)]
lib.mp_dsposv.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi, _pi]
lib.mp_dsposv_ex.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi, _pi, ctypes.POINTER(Opts), ctypes.POINTER(Report)]
lib.mp_dposv.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi]
lib.mp_dposv_ex.argtypes = [_i64, _i64, _p, _i64, _p, _p, _pi, ctypes.POINTER(Opts), ctypes.POINTER(Report)]
lib.mp_spotrf.argtypes = [_i64, _p, _i64, _p, _pi, ctypes.POINTER(Opts)]
lib.mp_dpotrf.argtypes = [_i64, _p, _i64, _p, _pi, ctypes.POINTER(Opts)]
lib.mp_qdgesv.argtypes = [_i64, _i64, _p, _i64, _p, _p, _p, _pi, _pi]
lib.mp_qdgesv_ex.argtypes = [_i64, _i64, _p, _i64, _p, _p, _p, _pi, _pi, ctypes.POINTER(Opts), ctypes.POINTER(Report)]
lib.mp_fgmres.argtypes = [_i64, _p, _i64, _p, _p, ctypes.c_int, ctypes.c_int, _pi, _pi]
lib.mp_fgmres_ex.argtypes = [_i64, _p, _i64, _p, _p, ctypes.c_int, ctypes.c_int, _pi, _pi, ctypes.POINTER(Opts),
                             ctypes.POINTER(Report)]
lib.mp_kernel_schur_update.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int]
lib.mp_kernel_schur_update_f64.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int]
lib.mp_set_stream.argtypes = [_p]
lib.mp_profile_collect.argtypes = [ctypes.POINTER(Report)]
lib.mp_last_error.restype = ctypes.c_char_p
lib.mp_version.restype = ctypes.c_char_p
lib.mp_exec_info.argtypes = [_pi, _pi, _pi]
lib.mp_get_unique_id.argtypes = [ctypes.c_char_p]
lib.mp_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_p)]
lib.mp_comm_init_loopback.argtypes = [ctypes.c_int, ctypes.POINTER(_p)]
lib.mp_comm_destroy.argtypes = [_p]
lib.mp_1dbc_local_cols.argtypes = [_i64, _i64, ctypes.c_int, ctypes.c_int]
lib.mp_1dbc_local_cols.restype = _i64
lib.mp_dsgesv_1dbc_ex.argtypes = [_p, _i64, _i64, _i64, _p, _i64, _p, _p, _pi, _pi, ctypes.POINTER(Opts),
                                  ctypes.POINTER(Report)]
lib.mp_dsgesv_1dbc.argtypes = [_p, _i64, _i64, _i64, _p, _i64, _p, _p, _pi, _pi]
lib.mp_dgesv_1dbc.argtypes = [_p, _i64, _i64, _i64, _p, _i64, _p, _p, _pi]

EXPORTED = ("mp_default_opts", "mp_dsgesv", "mp_dsgesv_ex", "mp_dgesv", "mp_dgesv_ex", "mp_sgetrf",
            "mp_dgetrf", "mp_set_stream", "mp_last_error", "mp_version", "mp_kernel_schur_update",
            "mp_kernel_schur_update_f64", "mp_dsposv", "mp_dsposv_ex", "mp_dposv", "mp_dposv_ex", "mp_spotrf",
            "mp_dpotrf", "mp_qdgesv", "mp_qdgesv_ex", "mp_fgmres", "mp_fgmres_ex",
            "mp_profile_collect", "mp_exec_info", "mp_get_unique_id", "mp_comm_init", "mp_comm_init_loopback",
            "mp_comm_destroy", "mp_1dbc_local_cols", "mp_dsgesv_1dbc", "mp_dsgesv_1dbc_ex", "mp_dgesv_1dbc")


def mp_version() -> str:
    return lib.mp_version().decode()


def _check(rc: int):
    if rc != MP_OK:
        raise MpError(f"libmpsolve error {rc}: {lib.mp_last_error().decode()}")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr_ld(M, name: str, square: bool, need_ld: int | None = None):
    """Pointer and leading dimension of a column-major float64 matrix (torch tensor or numpy array).

    The C-ABI reads B and X with leading dimension n (include/mp_solve.h), so callers pass
    ``need_ld=n`` for them: a row-sliced view (ld > n), a strided 1-D view or a non-float64
    array is rejected instead of being read (or written) as if it were contiguous."""
    if _is_torch(M):
        import torch
        if M.dtype != torch.float64:
            raise TypeError(f"{name} must be float64 (got {M.dtype})")
        if M.dim() == 1:
            if M.shape[0] > 1 and M.stride(0) != 1:
                raise ValueError(f"{name}: a 1-D view must be contiguous (stride 1)")
            ptr, ld = M.data_ptr(), max(M.shape[0], 1)
        elif M.dim() == 2:
            if M.shape[0] > 1 and M.shape[1] > 0 and M.stride(0) != 1:
                raise ValueError(f"{name} must be column-major (stride(0) == 1); use colmajor_cuda()")
            ptr, ld = M.data_ptr(), (M.stride(1) if M.shape[1] > 1 else max(M.shape[0], 1))
        else:
            raise ValueError(f"{name} must be 1-D or 2-D")
    else:
        A = np.asarray(M)
        if A.dtype != np.float64:
            raise TypeError(f"{name} must be float64 (got {A.dtype})")
        if A.ndim == 1:
            if not A.flags.c_contiguous:
                raise ValueError(f"{name}: a 1-D array must be contiguous")
        elif A.ndim == 2:
            if not A.flags.f_contiguous:
                raise ValueError(f"{name} must be Fortran-ordered (column-major, contiguous)")
        else:
            raise ValueError(f"{name} must be 1-D or 2-D")
        ptr, ld = A.ctypes.data, max(A.shape[0], 1)
    if need_ld is not None and ld != max(need_ld, 1):
        raise ValueError(f"{name} must have leading dimension n = {need_ld} (got {ld}); pass a contiguous copy")
    return ptr, ld


def _stream_of(*ts):
    for t in ts:
        if _is_torch(t) and t.is_cuda:
            import torch
            return torch.cuda.current_stream(t.device).cuda_stream
    return None


def colmajor_cuda(M, device="cuda"):
    """Fortran-ordered numpy (n, k) -> torch CUDA float64 tensor of shape (n, k), stride (1, n)."""
    import torch
    M = np.asfortranarray(np.asarray(M, dtype=np.float64))
    if M.ndim == 1:
        M = M[:, None]
    return torch.from_numpy(np.ascontiguousarray(M.T)).to(device).t()


def _alloc_like_X(B, n, nrhs):
    if _is_torch(B):
        import torch
        return torch.empty((nrhs, n), dtype=torch.float64, device=B.device).t()
    return np.zeros((n, nrhs), dtype=np.float64, order="F")


def _nrhs(B, n):
    return 1 if len(B.shape) == 1 else B.shape[1]


def mp_dsgesv_ex(A, B, X=None, opts: Opts | None = None, report: bool = True):
    """Mixed-precision solve; returns (X, iters, info, Report|None)."""
    n = A.shape[0]
    nrhs = _nrhs(B, n)
    if X is None:
        X = _alloc_like_X(B, n, nrhs)
    pa, lda = _ptr_ld(A, "A", True)
    pb, _ = _ptr_ld(B, "B", False, n)
    px, _ = _ptr_ld(X, "X", False, n)
    lib.mp_set_stream(_stream_of(A, B, X))
    it, info = ctypes.c_int(0), ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_dsgesv_ex(n, nrhs, pa, lda, pb, px, ctypes.byref(it), ctypes.byref(info),
                            ctypes.byref(opts) if opts is not None else None,
                            ctypes.byref(rep) if rep is not None else None))
    return X, it.value, info.value, rep


def mp_dsgesv(A, B, X=None, opts: Opts | None = None):
    X, it, info, _ = mp_dsgesv_ex(A, B, X, opts, report=False)
    return X, it, info


def mp_dgesv_ex(A, B, X=None, opts: Opts | None = None, report: bool = True):
    n = A.shape[0]
    nrhs = _nrhs(B, n)
    if X is None:
        X = _alloc_like_X(B, n, nrhs)
    pa, lda = _ptr_ld(A, "A", True)
    pb, _ = _ptr_ld(B, "B", False, n)
    px, _ = _ptr_ld(X, "X", False, n)
    lib.mp_set_stream(_stream_of(A, B, X))
    info = ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_dgesv_ex(n, nrhs, pa, lda, pb, px, ctypes.byref(info),
                           ctypes.byref(opts) if opts is not None else None,
                           ctypes.byref(rep) if rep is not None else None))
    return X, info.value, rep


def mp_dgesv(A, B, X=None, opts: Opts | None = None):
    X, info, _ = mp_dgesv_ex(A, B, X, opts, report=False)
    return X, info


def mp_dsposv_ex(A, B, X=None, opts: Opts | None = None, report: bool = True):
    """Mixed-precision SPD solve (lower triangle of A read); returns (X, iters, info, Report|None)."""
    n = A.shape[0]
    nrhs = _nrhs(B, n)
    if X is None:
        X = _alloc_like_X(B, n, nrhs)
    pa, lda = _ptr_ld(A, "A", True)
    pb, _ = _ptr_ld(B, "B", False, n)
    px, _ = _ptr_ld(X, "X", False, n)
    lib.mp_set_stream(_stream_of(A, B, X))
    it, info = ctypes.c_int(0), ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_dsposv_ex(n, nrhs, pa, lda, pb, px, ctypes.byref(it), ctypes.byref(info),
                            ctypes.byref(opts) if opts is not None else None,
                            ctypes.byref(rep) if rep is not None else None))
    return X, it.value, info.value, rep


def mp_dposv_ex(A, B, X=None, opts: Opts | None = None, report: bool = True):
    n = A.shape[0]
    nrhs = _nrhs(B, n)
    if X is None:
        X = _alloc_like_X(B, n, nrhs)
    pa, lda = _ptr_ld(A, "A", True)
    pb, _ = _ptr_ld(B, "B", False, n)
    px, _ = _ptr_ld(X, "X", False, n)
    lib.mp_set_stream(_stream_of(A, B, X))
    info = ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_dposv_ex(n, nrhs, pa, lda, pb, px, ctypes.byref(info),
                           ctypes.byref(opts) if opts is not None else None,
                           ctypes.byref(rep) if rep is not None else None))
    return X, info.value, rep


def mp_qdgesv_ex(A, B, Xhi=None, Xlo=None, opts: Opts | None = None, report: bool = True):
    """Extended-precision refinement (QDGESV analog): X = Xhi + Xlo (double-double);
    returns (Xhi, Xlo, iters, info, Report|None)."""
    n = A.shape[0]
    nrhs = _nrhs(B, n)
    if Xhi is None:
        Xhi = _alloc_like_X(B, n, nrhs)
    if Xlo is None:
        Xlo = _alloc_like_X(B, n, nrhs)
    pa, lda = _ptr_ld(A, "A", True)
    pb, _ = _ptr_ld(B, "B", False, n)
    ph, _ = _ptr_ld(Xhi, "Xhi", False, n)
    pl, _ = _ptr_ld(Xlo, "Xlo", False, n)
    lib.mp_set_stream(_stream_of(A, B, Xhi))
    it, info = ctypes.c_int(0), ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_qdgesv_ex(n, nrhs, pa, lda, pb, ph, pl, ctypes.byref(it), ctypes.byref(info),
                            ctypes.byref(opts) if opts is not None else None,
                            ctypes.byref(rep) if rep is not None else None))
    return Xhi, Xlo, it.value, info.value, rep


def mp_fgmres_ex(A, b, x=None, m_out: int = 10, m_in: int = 20, opts: Opts | None = None, report: bool = True):
    """Algorithm 2, FGMRES(m_out)-GMRES_SP(m_in) (include/mp_solve.h): returns (x, iters, info, Report|None)."""
    n = A.shape[0]
    if _nrhs(b, n) != 1:
        raise ValueError("mp_fgmres: one right-hand side")
    if x is None:
        x = _alloc_like_X(b, n, 1)
    pa, lda = _ptr_ld(A, "A", True)
    pb, _ = _ptr_ld(b, "b", False, n)
    px, _ = _ptr_ld(x, "x", False, n)
    lib.mp_set_stream(_stream_of(A, b, x))
    it, info = ctypes.c_int(0), ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_fgmres_ex(n, pa, lda, pb, px, int(m_out), int(m_in), ctypes.byref(it), ctypes.byref(info),
                            ctypes.byref(opts) if opts is not None else None,
                            ctypes.byref(rep) if rep is not None else None))
    return x, it.value, info.value, rep


def _potrf(fn, dtype, A, opts):
    n = A.shape[0]
    pa, lda = _ptr_ld(A, "A", True)
    L = np.zeros((n, n), dtype=dtype, order="F")
    info = ctypes.c_int(0)
    lib.mp_set_stream(_stream_of(A))
    _check(fn(n, pa, lda, L.ctypes.data, ctypes.byref(info), ctypes.byref(opts) if opts is not None else None))
    return L, info.value


def mp_spotrf(A, opts: Opts | None = None):
    """SPD step 1 alone (binary32 Cholesky of fl32(A)'s lower triangle): host (L Fortran, info)."""
    return _potrf(lib.mp_spotrf, np.float32, A, opts)


def mp_dpotrf(A, opts: Opts | None = None):
    return _potrf(lib.mp_dpotrf, np.float64, A, opts)


def _getrf(fn, dtype, A, opts):
    n = A.shape[0]
    pa, lda = _ptr_ld(A, "A", True)
    LU = np.zeros((n, n), dtype=dtype, order="F")
    ipiv = np.zeros(n, dtype=np.int32)
    info = ctypes.c_int(0)
    lib.mp_set_stream(_stream_of(A))
    _check(fn(n, pa, lda, LU.ctypes.data, ipiv.ctypes.data, ctypes.byref(info),
              ctypes.byref(opts) if opts is not None else None))
    return LU, ipiv, info.value


def mp_sgetrf(A, opts: Opts | None = None):
    """Step 1 alone (binary32 GEPP of fl32(A)); returns host (LU float32 Fortran, ipiv 0-based, info)."""
    return _getrf(lib.mp_sgetrf, np.float32, A, opts)


def mp_dgetrf(A, opts: Opts | None = None):
    return _getrf(lib.mp_dgetrf, np.float64, A, opts)


def mp_kernel_schur_update(W, r0: int, c0: int, k0: int, M: int, N: int, K: int, variant: int = MP_VARIANT_FFMA):
    """K5 alone on a row-major float32 CUDA tensor W (in place): W[r0:r0+M, c0:c0+N] -= W[r0:, k0:k0+K] @ W[k0:k0+K, c0:]."""
    if not (_is_torch(W) and W.is_cuda and W.element_size() == 4 and W.stride(1) == 1):
        raise TypeError("W must be a row-major float32 CUDA tensor")
    lib.mp_set_stream(_stream_of(W))
    _check(lib.mp_kernel_schur_update(W.data_ptr(), W.stride(0), r0, c0, k0, M, N, K, variant))


MP_F64_AUTO, MP_F64_DMMA, MP_F64_DFMA = 0, 1, 2


def mp_kernel_schur_update_f64(W, r0: int, c0: int, k0: int, M: int, N: int, K: int, pipe: int = MP_F64_AUTO):
    """The binary64 trailing update alone on a row-major float64 CUDA tensor W (in place)."""
    if not (_is_torch(W) and W.is_cuda and W.element_size() == 8 and W.stride(1) == 1):
        raise TypeError("W must be a row-major float64 CUDA tensor")
    lib.mp_set_stream(_stream_of(W))
    _check(lib.mp_kernel_schur_update_f64(W.data_ptr(), W.stride(0), r0, c0, k0, M, N, K, pipe))


def mp_profile_collect() -> Report:
    """Per-kernel-class totals of the calls made with flags 2|4 since the last collection."""
    rep = Report()
    _check(lib.mp_profile_collect(ctypes.byref(rep)))
    return rep


def make_opts(nb: int = 0, itermax: int = 30, variant: int = MP_VARIANT_3XTF32, flags: int = 0) -> Opts:
    o = Opts()
    lib.mp_default_opts(ctypes.byref(o))
    o.nb, o.itermax, o.variant, o.flags = nb, itermax, variant, flags
    return o


def mp_exec_info():
    """(lookahead, sms_panel, sms_update) of the factorisation on the current device."""
    la, sp, su = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    _check(lib.mp_exec_info(ctypes.byref(la), ctypes.byref(sp), ctypes.byref(su)))
    return la.value, sp.value, su.value


# --------------------------------------------------------------------------- multi-GPU (1D block-cyclic)
def local_columns(n: int, nb: int, nranks: int, rank: int) -> np.ndarray:
    """Global column indices owned by `rank` (increasing): block j lives on rank j % nranks."""
    nb = nb if nb > 0 else 256
    cols = [np.arange(j * nb, min(n, (j + 1) * nb)) for j in range(rank, -(-n // nb), nranks)]
    return np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)


def mp_1dbc_local_cols(n: int, nb: int, nranks: int, rank: int) -> int:
    return int(lib.mp_1dbc_local_cols(n, nb, nranks, rank))


def mp_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.mp_get_unique_id(buf))
    return buf.raw


def mp_comm_init(nranks: int, rank: int, uid: bytes):
    h = _p()
    _check(lib.mp_comm_init(nranks, rank, uid, ctypes.byref(h)))
    return h


def mp_comm_init_loopback(nranks: int):
    hs = (_p * nranks)()
    _check(lib.mp_comm_init_loopback(nranks, hs))
    return [_p(hs[r]) for r in range(nranks)]


def mp_comm_destroy(comm):
    _check(lib.mp_comm_destroy(comm))


def mp_dsgesv_1dbc_ex(comm, n: int, nb: int, A_local, B, X=None, opts: Opts | None = None, report: bool = True):
    """Distributed mixed-precision solve (collective).  A_local: this rank's columns (column-major CUDA
    tensor, n x local_cols); B, X replicated CUDA tensors (n x nrhs, column-major).  -> (X, iters, info, rep)."""
    nrhs = _nrhs(B, n)
    if X is None:
        X = _alloc_like_X(B, n, nrhs)
    nloc = A_local.shape[1] if len(A_local.shape) == 2 else 0
    pa, lda = _ptr_ld(A_local, "A_local", False) if nloc > 0 else (None, 1)
    pb, _ = _ptr_ld(B, "B", False, n)
    px, _ = _ptr_ld(X, "X", False, n)
    lib.mp_set_stream(_stream_of(B, X))
    it, info = ctypes.c_int(0), ctypes.c_int(0)
    rep = Report() if report else None
    _check(lib.mp_dsgesv_1dbc_ex(comm, n, nrhs, nb, pa, lda, pb, px, ctypes.byref(it), ctypes.byref(info),
                                 ctypes.byref(opts) if opts is not None else None,
                                 ctypes.byref(rep) if rep is not None else None))
    return X, it.value, info.value, rep


def mp_dgesv_1dbc(comm, n: int, nb: int, A_local, B, X=None):
    nrhs = _nrhs(B, n)
    if X is None:
        X = _alloc_like_X(B, n, nrhs)
    nloc = A_local.shape[1] if len(A_local.shape) == 2 else 0
    pa, lda = _ptr_ld(A_local, "A_local", False) if nloc > 0 else (None, 1)
    pb, _ = _ptr_ld(B, "B", False, n)
    px, _ = _ptr_ld(X, "X", False, n)
    lib.mp_set_stream(_stream_of(B, X))
    info = ctypes.c_int(0)
    _check(lib.mp_dgesv_1dbc(comm, n, nrhs, nb, pa, lda, pb, px, ctypes.byref(info)))
    return X, info.value
