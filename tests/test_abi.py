"""C-ABI checks that need no GPU: the library builds, loads and exports every
symbol include/mp_solve.h declares; argument validation (host logic) answers
before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binding():
    from paper_0808_2794_b200 import build
    build.build()
    from paper_0808_2794_b200 import binding as b
    return b


def header_functions():
    names = set()
    inc = os.path.join(ROOT, "include")
    for h in sorted(os.listdir(inc)):
        if h.endswith(".h"):
            txt = re.sub(r"/\*.*?\*/", "", open(os.path.join(inc, h)).read(), flags=re.S)
            names |= set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", txt))
    return sorted(names)


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("mp_dsgesv", "mp_dgesv", "mp_dsgesv_ex", "mp_dgesv_ex", "mp_sgetrf", "mp_dgetrf"):
        assert f in fns


def test_library_exports_every_declared_symbol(binding):
    for f in header_functions():
        assert hasattr(binding.lib, f), f
    assert set(header_functions()) == set(binding.EXPORTED)


def test_struct_layout_matches_header(binding):
    assert ctypes.sizeof(binding.Opts) == 16
    # 6 int32 + anrm + hist[64] + 6 doubles + 2 int64
    assert ctypes.sizeof(binding.Report) == 24 + 8 + 64 * 8 + 6 * 8 + 16 + 3 * 64


def test_version_and_defaults(binding):
    assert "sm_100a" in binding.mp_version()
    o = binding.Opts()
    binding.lib.mp_default_opts(ctypes.byref(o))
    assert (o.nb, o.itermax, o.variant, o.flags) == (0, 30, 1, 0)   # default variant: 3xTF32 tcgen05


def _call(binding, n, nrhs, A, lda, B, X):
    it, info = ctypes.c_int(7), ctypes.c_int(7)
    rc = binding.lib.mp_dsgesv(n, nrhs, A, lda, B, X, ctypes.byref(it), ctypes.byref(info))
    return rc, it.value, info.value


def test_argument_errors_without_device(binding):
    A = np.zeros((4, 4), order="F"); B = np.zeros((4, 1), order="F"); X = np.zeros((4, 1), order="F")
    pa, pb, px = A.ctypes.data, B.ctypes.data, X.ctypes.data
    assert _call(binding, -1, 1, pa, 4, pb, px)[0::2] == (0, -1)
    assert _call(binding, 4, -1, pa, 4, pb, px)[0::2] == (0, -2)
    assert _call(binding, 4, 1, None, 4, pb, px)[0::2] == (0, -3)
    assert _call(binding, 4, 1, pa, 3, pb, px)[0::2] == (0, -4)
    assert _call(binding, 4, 1, pa, 4, None, px)[0::2] == (0, -5)
    assert _call(binding, 4, 1, pa, 4, pb, None)[0::2] == (0, -6)
    assert _call(binding, 4, 1, pa, 4, pb, pa)[0::2] == (0, -6)          # X overlaps A
    assert _call(binding, 4, 1, pa, 4, pb, pb)[0::2] == (0, -6)          # X overlaps B
    assert _call(binding, 0, 1, pa, 1, pb, px) == (0, 0, 0)              # quick return
    assert _call(binding, 4, 0, pa, 4, pb, px) == (0, 0, 0)
    info = ctypes.c_int(7)
    assert binding.lib.mp_dgesv(-1, 1, pa, 4, pb, px, ctypes.byref(info)) == 0 and info.value == -1


def test_sass_is_sm100a(binding):
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_rejects_bad_layouts(binding):
    """B / X must have leading dimension n and be float64 (include/mp_solve.h); views that the
    C-ABI would misread are rejected before any call."""
    import torch
    n = 8
    A = torch.zeros((n, n), dtype=torch.float64).t()              # column-major
    big = torch.zeros((3, n + 4), dtype=torch.float64).t()         # (n+4, 3) stride (1, n+4)
    with pytest.raises(ValueError):
        binding._ptr_ld(big[:n], "B", False, n)                    # row-sliced: ld = n + 4 != n
    with pytest.raises(ValueError):
        binding._ptr_ld(torch.zeros(2 * n, dtype=torch.float64)[::2], "B", False, n)   # strided 1-D
    with pytest.raises(TypeError):
        binding._ptr_ld(torch.zeros((n, 1), dtype=torch.int64), "B", False, n)
    with pytest.raises(TypeError):
        binding._ptr_ld(np.zeros((n, 1), dtype=np.float32), "X", False, n)
    with pytest.raises(ValueError):
        binding._ptr_ld(np.zeros((n, 3)), "X", False, n)           # C-ordered 2-D
    assert binding._ptr_ld(A, "A", True)[1] == n
    assert binding._ptr_ld(torch.zeros((2, n), dtype=torch.float64).t(), "B", False, n)[1] == n
    assert binding._ptr_ld(np.zeros(n), "B", False, n)[1] == n
