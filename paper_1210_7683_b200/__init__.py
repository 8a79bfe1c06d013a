"""B200-native GLS-grid engine (arXiv 1210.7683 hot path), drop-in for gwgrid.

The m x t grid of GLS problems b_ij = (X_i^T M_j^-1 X_i)^-1 X_i^T M_j^-1 y_j,
solved after the one-off CPU eigendecomposition of the kinship matrix, runs on
the GPU: a deterministic DMMA rotation kernel, a per-trait context kernel, and a fused
FP64-DMMA grid kernel with the p x p Cholesky solves in its epilogue.
"""
from .engine import (Engine, device_working_set_bytes, eigendecompose, solve_cell, solve_grid,
                     verify_grid)
from .errors import (BackendError, DeviceError, DimensionError, GwgridError,
                     InfeasibleBudgetError, IoError, NonSymmetricError, NotPositiveDefiniteError)

__all__ = [
    "Engine", "eigendecompose", "solve_grid", "solve_cell", "verify_grid",
    "device_working_set_bytes",
    "GwgridError", "DimensionError", "NonSymmetricError", "BackendError",
    "NotPositiveDefiniteError", "IoError", "InfeasibleBudgetError", "DeviceError",
]

__version__ = "0.1.0"
