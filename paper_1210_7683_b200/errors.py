"""Exception hierarchy mirroring gwgrid's (proj/include/gwgrid/types.hpp:34-94).

The reference's Python layer maps NotPositiveDefinite / Dimension /
NonSymmetric / InfeasibleBudget to ValueError, IoError to OSError and other
errors to RuntimeError (proj/python/bindings.cpp:232-248); these classes keep
that mapping (they subclass the same builtins) and add the typed coordinates.
"""
from __future__ import annotations

from . import _native as nat


class GwgridError(Exception):
    """Base of every error raised by the engine."""


class DimensionError(GwgridError, ValueError):
    pass


class NonSymmetricError(GwgridError, ValueError):
    pass


class BackendError(GwgridError, RuntimeError):
    pass


class NotPositiveDefiniteError(GwgridError, ValueError):
    def __init__(self, msg: str, snp_index: int = -1, trait_index: int = -1):
        super().__init__(msg)
        self.snp_index = snp_index
        self.trait_index = trait_index


class IoError(GwgridError, OSError):
    pass


class InfeasibleBudgetError(GwgridError, ValueError):
    pass


class DeviceError(GwgridError, RuntimeError):
    """CUDA runtime / device failure (no reference analogue)."""


def raise_for(st: "nat.Status") -> None:
    code = st.code
    if code == nat.GWG_OK:
        return
    msg = st.msg.decode(errors="replace")
    if code == nat.GWG_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefiniteError(msg, st.snp_index, st.trait_index)
    cls = {
        nat.GWG_DIMENSION: DimensionError,
        nat.GWG_NON_SYMMETRIC: NonSymmetricError,
        nat.GWG_BACKEND: BackendError,
        nat.GWG_IO: IoError,
        nat.GWG_INFEASIBLE_BUDGET: InfeasibleBudgetError,
        nat.GWG_CUDA: DeviceError,
    }.get(code, GwgridError)
    raise cls(msg)
