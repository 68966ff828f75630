"""Exception types of the reference API, defined once and re-exported by the
modules that own them in the reference:

    ModeError           precision.py:27-28
    AssemblyError       tensor.py:21-22
    KernelError         kernels.py:27-28
    NormalizationError  kernels.py:31-32
    CollectiveError     comm.py:30-31
    CollectiveTimeout   comm.py:34-41
    ContractError       hopm.py:32-33
"""

from __future__ import annotations


class ModeError(ValueError):
    """Unknown precision mode or invalid storage/compute combination."""


class AssemblyError(ValueError):
    """Subtensors do not belong to the given split plan."""


class KernelError(ValueError):
    """Shape mismatch or invalid kernel arguments."""


class NormalizationError(ArithmeticError):
    """Attempt to normalize a zero vector."""


class CollectiveError(RuntimeError):
    """Mismatched participation in a collective."""


class CollectiveTimeout(CollectiveError):
    """A collective gave up waiting; reports which ranks never arrived."""

    def __init__(self, kind: str, absent: list[int]):
        self.kind = kind
        self.absent = absent
        super().__init__(f"collective {kind!r} timed out waiting for ranks {absent}")


class ContractError(ValueError):
    """Distributed operands do not fit the requested contraction."""


class DeviceError(RuntimeError):
    """CUDA runtime failure inside libtenvec_b200 (error code 5)."""
