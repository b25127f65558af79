"""Error taxonomy of the B200 engine.

Mirrors the reference's exception classes (convkit ``errors.py:8-37``) so a
caller that catches ``convkit.errors.ConfigError`` semantics gets the same
type here, and maps the C-ABI status codes of ``include/ckb200.h`` onto them.
"""

from __future__ import annotations


class ConvkitError(Exception):
    """Root of every error raised by this package."""


class DimensionError(ConvkitError):
    """Shapes or map counts disagree."""


class GeometryError(ConvkitError):
    """Impossible layer geometry (kernel bigger than map, size < 1, ...)."""


class ConfigError(ConvkitError):
    """Bad configuration value or malformed architecture text."""


class DataFormatError(ConvkitError):
    """Malformed dataset content."""


class StateError(ConvkitError):
    """Call made against missing or stale runtime state."""


class PrecisionError(ConvkitError):
    """The B200 path computes in FP32 only; double nets stay on the CPU."""


class GeometryWarning(UserWarning):
    """Legal but lossy geometry (fractional placement, pool truncation)."""


class CudaError(ConvkitError):
    """The CUDA runtime reported a failure inside the native library."""


# status codes returned by every ck_* entry point (include/ckb200.h)
CK_OK = 0
CK_E_DIMENSION = -1
CK_E_GEOMETRY = -2
CK_E_CONFIG = -3
CK_E_STATE = -4
CK_E_PRECISION = -5
CK_E_CUDA = -6
CK_E_NOMEM = -7

_BY_CODE = {
    CK_E_DIMENSION: DimensionError,
    CK_E_GEOMETRY: GeometryError,
    CK_E_CONFIG: ConfigError,
    CK_E_STATE: StateError,
    CK_E_PRECISION: PrecisionError,
    CK_E_CUDA: CudaError,
    CK_E_NOMEM: CudaError,
}


def error_for_status(code: int, message: str) -> ConvkitError:
    """Exception instance for a non-zero ck_* status."""
    return _BY_CODE.get(code, ConvkitError)(f"[ck status {code}] {message}")
