"""Exception hierarchy of the drop-in host API.

Same class names and inheritance as the reference package
(/root/reference/pkg/src/ptsbe/errors.py:4-38) so that callers' `except`
clauses keep working.  `DeviceError` is new: it is raised when the CUDA
library is missing or a CUDA call fails (there is no CPU fallback).
"""


class SimulationError(Exception):
    """Root of every error this package raises on purpose."""


class NetworkStructureError(SimulationError):
    """Malformed tensor network or contraction step."""


class IncompletePathError(NetworkStructureError):
    """Path replay ended with more than one operand left."""


class CapacityError(SimulationError):
    """Input is beyond a hard size cap of the component asked to handle it."""


class ResourceLimitError(SimulationError):
    """Intermediate-size ceiling or wall-clock deadline tripped."""


class PathCacheError(SimulationError):
    """A stored path does not replay on a network with the same signature."""


class ImpossiblePrefixError(SimulationError):
    """Conditional marginal has (numerically) zero total mass."""


class NumericalError(SimulationError):
    """Marginal diagonal entry below the negative tolerance."""


class DeviceError(SimulationError):
    """libptsbe_b200.so missing / not loadable, or a CUDA runtime failure."""


# C-ABI status codes (include/ptsbe_b200.h) -> exception classes.
STATUS_TO_ERROR = {
    1: ValueError,
    2: NetworkStructureError,
    3: ResourceLimitError,
    4: NumericalError,
    5: ImpossiblePrefixError,
    6: DeviceError,
    7: CapacityError,
}
