"""Exception taxonomy mirroring the reference's (errors.py:4-53), so callers
catch the same classes.  Device status codes map onto them in _raise()."""


class FuseoptError(Exception):
    """Base class for all package errors."""


class CycleError(FuseoptError):
    """The contracted or scheduling dependency graph contains a cycle."""


class MissingCost(FuseoptError):
    """A group or bucket has no duration available."""


class NotNeighbors(FuseoptError):
    """AllReduce fusion between non-neighbouring buckets."""


class UnknownOp(FuseoptError, KeyError):
    """Profile lookup missed."""


class DimensionMismatch(FuseoptError):
    """Model parameters and feature dimensions disagree."""


class LimitExceeded(FuseoptError):
    """Exhaustive enumeration above its size limits."""


class InvalidConfig(FuseoptError):
    """Search configuration violates its invariants."""


class GraphFormatError(FuseoptError, ValueError):
    """A graph/profile/model document does not match the expected schema."""


class DeviceError(FuseoptError, RuntimeError):
    """CUDA runtime failure or a configuration outside the device path."""


def _raise(status: int, what: str, detail: str = "") -> None:
    """Map an fo_status code (include/disco_b200.h) to the reference's class."""
    from . import _native as N

    msg = f"{what}: {detail}" if detail else what
    if status == N.FO_OK:
        return
    if status == N.FO_CYCLE:
        raise CycleError(msg)
    if status == N.FO_MISSING_COST:
        raise MissingCost(msg)
    if status == N.FO_NEGATIVE_DURATION:
        raise ValueError(msg)
    if status == N.FO_DIM_MISMATCH:
        raise DimensionMismatch(msg)
    if status == N.FO_INVALID_ARG:
        raise GraphFormatError(msg)
    raise DeviceError(f"{msg} (status {status})")
