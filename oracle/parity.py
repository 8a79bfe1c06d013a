"""Parity metrics of a device grid against the oracle's — TEST INFRASTRUCTURE.

Used by tests/ and by bench.py's cpu_baseline leg (whose oracle grid is the
reference).  BASELINE.json's north star asks for a max component-wise
relative error of 1e-8; the reference's own verify metric is norm-wise per
cell (proj/tools/gwgrid_main.cpp:378-380).  Components whose exact value is
~0 have no meaningful relative error under any two rounding orders (SURVEY.md
§7), so three numbers are reported: norm-wise, component-wise floored at 1e-6
of the cell norm, and the raw component-wise maximum with the count of
components above 1e-8.
"""
from __future__ import annotations

import numpy as np

NORMWISE_TOL = 1e-10
COMPONENT_TOL = 1e-8


def parity_metrics(got: np.ndarray, ref: np.ndarray, chunk: int = 4096) -> dict:
    """North-star parity of a whole grid against the oracle's:
    norm-wise per cell (the reference's verify metric), component-wise
    floored at 1e-6 of the cell norm, and the raw component-wise maximum with
    the count of components above 1e-8."""
    normwise = floored = raw = 0.0
    over = comps = 0
    worst = None
    with np.errstate(divide="ignore", invalid="ignore"):
        for a in range(0, got.shape[0], chunk):
            g, r = got[a:a + chunk], ref[a:a + chunk]
            d = np.abs(g - r)
            nrm = np.linalg.norm(r, axis=-1)
            normwise = max(normwise, float((np.linalg.norm(g - r, axis=-1) / nrm).max()))
            floored = max(floored, float((d / np.maximum(np.abs(r), 1e-6 * nrm[..., None])).max()))
            rel = np.where(d == 0, 0.0, d / np.abs(r))
            k = int(np.argmax(rel))
            if rel.flat[k] > raw:
                raw = float(rel.flat[k])
                worst = {"abs_ref": float(np.abs(r).flat[k]),
                         "cell_norm": float(nrm.flat[k // r.shape[-1]])}
            over += int((rel > 1e-8).sum())
            comps += rel.size
    return {"cells": int(np.prod(got.shape[:-1])), "components": comps,
            "normwise_max": normwise, "floored_componentwise_max": floored,
            "raw_componentwise_max": raw, "n_raw_over_1e-8": over, "raw_max_at": worst,
            "tolerance": {"normwise": NORMWISE_TOL, "floored_componentwise": COMPONENT_TOL},
            "pass": bool(normwise <= NORMWISE_TOL and floored <= COMPONENT_TOL),
            "reference": "oracle/ compute_grid (restated gwgrid compute_tile) on the same inputs"}
