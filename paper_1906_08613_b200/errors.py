"""Error classes of the backend, mirroring the reference's hierarchy
(/root/reference/pkg/src/lagen/errors.py:4-59).

When the reference package `lagen` is importable, the classes below subclass
its own `LagenError` / `VerificationError`, so callers of the reference API
(`except VerificationError`) catch backend failures unchanged.  Exit-code
mapping stays the reference's (cli.py:385-406): VerificationError -> 1,
other LagenError -> 2.
"""

try:  # pragma: no cover - depends on the environment
    from lagen.errors import LagenError as _RefLagenError
    from lagen.errors import VerificationError as _RefVerificationError
except Exception:  # reference not installed: same names, standalone
    class _RefLagenError(Exception):
        """Base class for all generator errors."""

    class _RefVerificationError(_RefLagenError):
        """Numeric verification failed (residual above tolerance, NaN, ...)."""


class LagenError(_RefLagenError):
    """Base class for backend errors (reference: errors.py:4-5)."""


class VerificationError(LagenError, _RefVerificationError):
    """Non-positive pivot or NaN/Inf in a solve (kernels.py:87-88, verify.py:301-302)."""


class UsageError(LagenError, ValueError):
    """Bad arguments (reference: cli.UsageError, exit code 2)."""


class UnsupportedSizeError(UsageError):
    """(n, b) has no sm_100a instance or b does not divide n."""


class VariantError(UsageError):
    """A statement list the backend cannot execute."""


class DeviceError(LagenError, RuntimeError):
    """CUDA runtime failure."""
