"""Order-independent result checksum, host side.

The device accumulates, for every cell (i, j) and component c it solves with
``checksum=True``, the term ``mix64((key(i, j) + c*K3) ^ bits(b_ijc))`` with
``key(i, j) = mix64(i*K1 + j*K2)`` into a wrapping uint64 sum
(csrc/slab_kernels.cuh, ``gwg_cell_hash`` in the C ABI).  A sum of per-component
terms does not depend on slab width, layout, shard split or GPU count, so one
64-bit number certifies a 3.2 TB grid (BASELINE config 3) against any other
run of it.  This module recomputes it from a downloaded grid (numpy, chunked)
so tests can tie the device checksum to actual bits.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_KI = np.uint64(0xD1B54A32D192ED03)
_KJ = np.uint64(0xA24BAED4963EE407)
_KC = np.uint64(0x9FB21C651E98DF25)
_S30, _S27, _S31 = np.uint64(30), np.uint64(27), np.uint64(31)


def _mix(x: np.ndarray) -> np.ndarray:
    x = x + _M0
    x = (x ^ (x >> _S30)) * _M1
    x = (x ^ (x >> _S27)) * _M2
    return x ^ (x >> _S31)


def grid_checksum(b: np.ndarray, i0: int = 0, layout: str = "numpy", chunk: int = 4096) -> int:
    """Checksum of a result grid: ``b`` is (m, t, p) for layout "numpy" or
    (t, m, p) for "stream"; SNP i of the grid is global index i0 + i."""
    b = np.asarray(b, dtype=np.float64)
    if layout == "stream":
        b = b.transpose(1, 0, 2)
    m, t, p = b.shape
    total = np.uint64(0)
    jj = np.arange(t, dtype=np.uint64)[None, :]
    cc = (np.arange(p, dtype=np.uint64) * _KC)[None, None, :]
    with np.errstate(over="ignore"):
        for a in range(0, m, chunk):
            blk = np.ascontiguousarray(b[a:a + chunk])
            ii = (np.arange(a, a + blk.shape[0], dtype=np.uint64) + np.uint64(i0))[:, None]
            key = _mix(ii * _KI + jj * _KJ)[:, :, None]
            terms = _mix((key + cc) ^ blk.view(np.uint64))
            total = total + terms.sum(dtype=np.uint64)
    return int(total)
