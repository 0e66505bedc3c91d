"""Exception types mirroring the reference's (and the C-ABI status codes).

Reference: DimensionMismatch (sparse.hpp:25-27), DegenerateDirection
(condest.hpp:35-37), StructurallySingular / NumericallySingular (lu.hpp:24-40),
ZeroRHS / ZeroSolution (error_bounds.hpp:33-39). ``std::invalid_argument`` and
``std::logic_error`` map onto ValueError subclasses / LogicError.
"""
from __future__ import annotations


class CondkitError(Exception):
    status = -1


class DimensionMismatch(CondkitError, ValueError):
    status = 1


class InvalidArgument(CondkitError, ValueError):
    status = 2


class LogicError(CondkitError, RuntimeError):
    status = 3


class StructurallySingular(CondkitError, RuntimeError):
    status = 4

    def __init__(self, msg: str = "", column: int = -1):
        super().__init__(msg)
        self.column = column


class NumericallySingular(CondkitError, RuntimeError):
    status = 5

    def __init__(self, msg: str = "", column: int = -1, pivot: float = 0.0):
        super().__init__(msg)
        self.column = column
        self.pivot = pivot


class ZeroRHS(InvalidArgument):
    status = 6


class ZeroSolution(InvalidArgument):
    status = 7


class ZeroColumn(CondkitError, RuntimeError):
    """column_scale on an empty or zero-norm column (sparse.hpp:29-33)."""
    status = 8

    def __init__(self, msg: str = "", column: int = -1):
        super().__init__(msg)
        self.column = column


class ZeroRow(CondkitError, RuntimeError):
    """row_scale on a zero-norm row (sparse.hpp:35-39)."""
    status = 9

    def __init__(self, msg: str = "", row: int = -1):
        super().__init__(msg)
        self.row = row


class CudaError(CondkitError, RuntimeError):
    status = 20


class DeviceUnavailable(CondkitError, RuntimeError):
    status = 21


class Unsupported(CondkitError, RuntimeError):
    status = 22


class DeviceOutOfMemory(CondkitError, MemoryError):
    status = 23


class NativeLibraryMissing(CondkitError, ImportError):
    status = -2


class DegenerateDirection(CondkitError, RuntimeError):
    """Operator maps the direction to zero (condest.hpp:35-37)."""


_BY_STATUS = {c.status: c for c in (DimensionMismatch, InvalidArgument, LogicError,
                                     StructurallySingular, NumericallySingular, ZeroRHS,
                                     ZeroSolution, ZeroColumn, ZeroRow, CudaError,
                                     DeviceUnavailable, Unsupported,
                                     DeviceOutOfMemory)}


def from_status(status: int, msg: str) -> CondkitError:
    cls = _BY_STATUS.get(status, CondkitError)
    if "DegenerateDirection" in msg:
        return DegenerateDirection(msg)
    return cls(msg)
