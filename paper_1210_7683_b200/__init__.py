"""B200-native GLS-grid engine (arXiv 1210.7683 hot path), drop-in for gwgrid.

The m x t grid of GLS problems b_ij = (X_i^T M_j^-1 X_i)^-1 X_i^T M_j^-1 y_j,
solved after the one-off CPU eigendecomposition of the kinship matrix, runs on
the GPU through the C ABI of include/gwgrid_cuda.h:

* genotype-coded SNP slabs (BASELINE.json's X_R in {0, 1, 2}; the default
  path): the rotation X'.X' exactly on the int8 tensor cores (tcgen05, seven
  8-bit slices of Z), S_BR on the FP64 tensor pipe (DMMA) through a positive
  exponential-sum factorisation of the GLS weights, and the p linear terms
  exactly on int8 tcgen05 fused with the bordered Cholesky solve and the
  store of b_ij (linear_solve_kernel);
* real-valued SNP slabs: a deterministic DMMA rotation and a fused FP64-DMMA
  grid kernel with the p x p Cholesky solves in its epilogue.

Slabs stream from host memory (float64 or int8 codes) through a
double-buffered H2D / compute / D2H pipeline into a host array or a result
sink; a device Group shards the SNP axis over several GPUs.
"""
from .checksum import grid_checksum
from .engine import (Engine, Group, device_working_set_bytes, eigendecompose, solve_cell,
                     solve_grid, verify_grid)
from .errors import (BackendError, DeviceError, DimensionError, GwgridError,
                     InfeasibleBudgetError, IoError, NonSymmetricError, NotPositiveDefiniteError)

__all__ = [
    "Engine", "Group", "eigendecompose", "solve_grid", "solve_cell", "verify_grid",
    "device_working_set_bytes", "grid_checksum",
    "GwgridError", "DimensionError", "NonSymmetricError", "BackendError",
    "NotPositiveDefiniteError", "IoError", "InfeasibleBudgetError", "DeviceError",
]

__version__ = "0.2.0"
