"""Exception types of the drop-in API.

Same names, hierarchy and meaning as the reference's
``pkg/src/leorzf/errors.py:8-54``.  When the reference package is installed
(``import leorzf`` works), every class here also SUBCLASSES the reference's
class of the same name, so a caller that catches ``leorzf.errors.X`` -- the
reference's CLI and harness (cli.py:290-299) -- catches what this package
raises after the swap INTEGRATION.md shows.

Device kernels never raise: they write a per-item status code into an
``int32 info[B]`` array (see ``include/leorzf_b200.h``) and the Python
layer maps the codes below onto these exceptions for single-item calls.
"""


try:  # the reference installed: be its exception classes too
    from leorzf import errors as _ref
except Exception:  # pragma: no cover - depends on the environment
    _ref = None


def _also(name: str) -> tuple:
    """(the reference's class of that name,) when it is importable."""
    return (getattr(_ref, name),) if _ref is not None and hasattr(_ref, name) else ()


class ConfigError(*(_also("ConfigError") or (Exception,))):
    """Invalid scenario configuration (reference errors.py:8)."""


class ParseError(ConfigError, *_also("ParseError")):
    """Config text could not be parsed (reference errors.py:12)."""


class UnknownKeyError(ConfigError, *_also("UnknownKeyError")):
    """Unknown configuration key (reference errors.py:16)."""


class RangeError(ConfigError, *_also("RangeError")):
    """Configuration value out of range (reference errors.py:20)."""


class SimulationError(*(_also("SimulationError") or (Exception,))):
    """Numerical failure while running the precoder update (errors.py:24)."""


class DimensionMismatchError(SimulationError, *_also("DimensionMismatchError")):
    """Operands have incompatible shapes (errors.py:28)."""


class SingularMatrixError(SimulationError, *_also("SingularMatrixError")):
    """Condition estimate above 1e14 or non-finite (errors.py:32)."""


class SingularAuxiliaryError(SimulationError, *_also("SingularAuxiliaryError")):
    """Woodbury r x r auxiliary matrix condition above 1e12 (errors.py:36)."""


class UnsupportedGeometryError(SimulationError, *_also("UnsupportedGeometryError")):
    """Array geometry outside what an operation supports (errors.py:41)."""


class BelowMinElevationError(SimulationError, *_also("BelowMinElevationError")):
    """A served user terminal is below the elevation mask (errors.py:45)."""


class ZeroPrecoderError(SimulationError, *_also("ZeroPrecoderError")):
    """Precoder has zero Frobenius norm (errors.py:49)."""


class EmptyInputError(SimulationError, *_also("EmptyInputError")):
    """Operation requires a non-empty input (errors.py:53)."""


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing, was built for another target, or a
    launch failed. There is deliberately no CPU fallback."""


# Per-item status codes written by the kernels (include/leorzf_b200.h).
INFO_OK = 0
INFO_SINGULAR = 1            # not PD / cond > 1e14 / non-finite  -> SingularMatrixError
INFO_SINGULAR_AUX = 2        # cond(aux) > 1e12                    -> SingularAuxiliaryError
INFO_ZERO_PRECODER = 3       # ||F_RF F_raw||_F == 0              -> ZeroPrecoderError
INFO_INDEFINITE = 4          # Hermitian, not PD, inverted by the pivoted path (not an error)
