"""Exception contract of the rasterizer boundary.

Same class names and base classes as the reference's error module
(`/root/reference/pkg/src/slimsplat/errors.py:4-37`) so callers that catch the
reference's exceptions keep working after the swap.  Status codes returned by
the C-ABI (`include/tgs.h`, `TGS_ERR_*`) are mapped onto these classes by
`raise_for_status`.
"""

from __future__ import annotations


class SlimsplatError(Exception):
    """Base class for all package errors (errors.py:4)."""


class DegenerateRotationError(SlimsplatError, ValueError):
    """Quaternion with (near-)zero norm (errors.py:8; geometry.py:23-24)."""


class SingularCovarianceError(SlimsplatError, ValueError):
    """2D covariance not positive definite (errors.py:12)."""


class ContractViolationError(SlimsplatError, ValueError):
    """Inputs violate a precondition (errors.py:16)."""


class EmptySceneError(SlimsplatError, ValueError):
    """A scene with no Gaussians where one is required (errors.py:20)."""


class DivergenceError(SlimsplatError, RuntimeError):
    """Non-finite loss; carries a diagnostic snapshot (errors.py:32-37)."""

    def __init__(self, message: str, snapshot: dict | None = None):
        super().__init__(message)
        self.snapshot = snapshot or {}


class NativeLibraryError(SlimsplatError, RuntimeError):
    """The CUDA library is missing, failed to load, or a CUDA call failed."""


# status codes of include/tgs.h
TGS_OK = 0
TGS_ERR_INVALID = 1
TGS_ERR_DEGENERATE_ROTATION = 2
TGS_ERR_CUDA = 3
TGS_ERR_UNSUPPORTED = 4
TGS_ERR_CAPACITY = 5


def raise_for_status(code: int, what: str) -> None:
    if code == TGS_OK:
        return
    if code == TGS_ERR_INVALID or code == TGS_ERR_UNSUPPORTED:
        raise ContractViolationError(f"{what}: invalid argument (status {code})")
    if code == TGS_ERR_DEGENERATE_ROTATION:
        raise DegenerateRotationError("quaternion with (near-)zero norm")
    if code == TGS_ERR_CAPACITY:
        raise NativeLibraryError(f"{what}: buffer capacity exceeded")
    raise NativeLibraryError(f"{what}: CUDA failure (status {code})")
