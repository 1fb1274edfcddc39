"""Error model mirroring parfrac::Errc / parfrac::Error (proj/core/include/parfrac/error.hpp:8-44).

The ordinals are the C-ABI return codes (include/pf_b200.h, PF_*), offset by one
so that 0 means success.
"""
from __future__ import annotations

import enum


class Errc(enum.IntEnum):
    DuplicateShift = 0
    LengthMismatch = 1
    UnderDetermined = 2
    UnknownMethod = 3
    InvalidFunction = 4
    NonUnitConstant = 5
    SingularShift = 6
    ZeroPivot = 7
    OutOfConvergenceRadius = 8
    BadArgument = 9
    # not in the reference: device-side failures of the B200 runtime
    CudaError = 10


class PfError(RuntimeError):
    """parfrac::Error: code + message; is_numerical() -> CLI exit 3 (error.hpp:29-38)."""

    def __init__(self, code: Errc, what: str):
        super().__init__(what)
        self.code = Errc(code)

    def is_numerical(self) -> bool:
        return self.code in (Errc.SingularShift, Errc.ZeroPivot, Errc.OutOfConvergenceRadius)


def raise_error(code: Errc, what: str):
    raise PfError(code, what)
