"""Error taxonomy of the B200 engine.

Mirrors the reference's exception classes (convkit ``errors.py:8-37``) and
maps the C-ABI status codes of ``include/ckb200.h`` onto them.

When the reference package ``convkit`` is importable (the drop-in case: the
reference's own code calls into this engine), every class here also derives
from its ``convkit.errors`` namesake, so ``except convkit.errors.ConfigError``
catches what this engine raises.  ``CK_STANDALONE_ERRORS=1`` opts out (and
avoids importing convkit, which pulls in numba).
"""

from __future__ import annotations

import importlib.util
import os


def _reference_errors():
    if os.environ.get("CK_STANDALONE_ERRORS") == "1":
        return None
    try:
        if importlib.util.find_spec("convkit") is None:
            return None
        import convkit.errors as ref
    except Exception:        # a broken or partial install: stay standalone
        return None
    return ref


_REF = _reference_errors()


def _bases(name, own):
    """(own,) plus the reference class of the same name when available."""
    ref = getattr(_REF, name, None) if _REF is not None else None
    if ref is None or issubclass(own, ref):
        return (own,)
    return (ref,) if issubclass(ref, own) else (own, ref)


class ConvkitError(*_bases("ConvkitError", Exception)):
    """Root of every error raised by this package."""


class DimensionError(*_bases("DimensionError", ConvkitError)):
    """Shapes or map counts disagree."""


class GeometryError(*_bases("GeometryError", ConvkitError)):
    """Impossible layer geometry (kernel bigger than map, size < 1, ...)."""


class ConfigError(*_bases("ConfigError", ConvkitError)):
    """Bad configuration value or malformed architecture text."""


class DataFormatError(*_bases("DataFormatError", ConvkitError)):
    """Malformed dataset content."""


class StateError(*_bases("StateError", ConvkitError)):
    """Call made against missing or stale runtime state."""


class PrecisionError(*_bases("PrecisionError", ConvkitError)):
    """The B200 path computes in FP32 only; double nets stay on the CPU."""


class GeometryWarning(*_bases("GeometryWarning", UserWarning)):
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
