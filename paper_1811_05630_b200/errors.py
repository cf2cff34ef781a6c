"""Exception taxonomy -- mirror of proj/include/qcsim/errors.hpp:21-53.

std::invalid_argument maps to ValueError; status codes come from the C-ABI
(include/qcsim_c.h, qcsim_status).
"""
from __future__ import annotations


class QcsimError(RuntimeError):
    pass


class CodecError(QcsimError):
    """Malformed or truncated compressed-block data (errors.hpp:24-27)."""


class ParseError(QcsimError):
    """Circuit-text syntax error with the 1-based line (errors.hpp:30-39)."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


class CapacityError(QcsimError):
    """Dense-materialization guard exceeded (errors.hpp:42-45)."""


class NumericError(QcsimError):
    """Norm drift beyond tolerance (errors.hpp:48-51)."""


class CudaError(QcsimError):
    """CUDA runtime failure (no reference analogue; there is no CPU fallback)."""


def raise_status(rc: int, lib) -> None:
    if rc == 0:
        return
    msg = lib.qcsim_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise CodecError(msg)
    if rc == 3:
        raise CapacityError(msg)
    if rc == 4:
        raise ParseError(0, msg)
    if rc == 5:
        raise NumericError(msg)
    if rc == 6:
        raise CudaError(msg)
    if rc == 7:
        raise MemoryError(msg)
    raise QcsimError(msg)
