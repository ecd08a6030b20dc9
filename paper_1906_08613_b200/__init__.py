"""B200-native execution backend for the `lagen` blocked-variant solvers
(arXiv 1906.08613): batched fp64 upper Cholesky, triangular Lyapunov and
triangular Sylvester on sm_100a.

The reference frontend (equation -> PME -> invariants -> blocked variants)
stays the reference's; this package replaces its executor
(verify.interpret_algorithm / the emitted C kernels) with CUDA kernels behind
the C ABI in include/lagen_b200.h.
"""

from . import errors, variants
from .variants import EQUATIONS, builtin_variants, default_blocks

__all__ = ["errors", "variants", "EQUATIONS", "builtin_variants", "default_blocks",
           "solve", "solve_host", "execute_batched", "interpret_algorithm", "generate",
           "load"]


def load():
    """Load the kernel library (raises ImportError if it was not built)."""
    from . import _lib
    return _lib


def __getattr__(name):
    if name in ("solve", "solve_host", "execute_batched", "interpret_algorithm", "generate"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
