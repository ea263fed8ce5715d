"""paper_0808_2794_b200 — B200-native mixed-precision iterative-refinement solver.

The hot path of arXiv 0808.2794 Alg. 1 with BASELINE.json's
stop test: FP32 blocked GEPP + FP32 triangular solves + FP64 residual/update on
sm_100a, behind the C-ABI of include/mp_solve.h (libmpsolve.so).  This package
is the thin Python binding (argument marshalling only) plus input generators.
"""
import importlib

from .inputs import BASE_SEED  # noqa: F401  (input generators carry no method arithmetic)

_SUBMODULES = {"binding", "build", "inputs"}


def __getattr__(name):
    # lazy: importing the package (e.g. for inputs) must not require the CUDA library
    if name.startswith("_") or name in _SUBMODULES:
        raise AttributeError(name)
    binding = importlib.import_module(__name__ + ".binding")
    try:
        return getattr(binding, name)
    except AttributeError:
        raise AttributeError(name) from None
