"""Parity metrics of a device grid against the oracle's — TEST INFRASTRUCTURE.

Used by tests/ and by bench.py's cpu_baseline leg (whose oracle grid is the
reference).  BASELINE.json's north star asks for a max component-wise
relative error of 1e-8; the reference's own verify metric is norm-wise per
cell (proj/tools/gwgrid_main.cpp:378-380).  Components whose exact value is
~0 have no meaningful relative error under any two rounding orders (SURVEY.md
§7), so three numbers are reported: norm-wise, component-wise floored at 1e-6
of the cell norm, and the raw component-wise maximum with the count of
components above 1e-8 (a component near zero has no meaningful relative
error: the asserted component-wise bound is allclose(rtol=1e-8,
atol=1e-13 |b_cell|), reported as the 1e-5-floored metric).
"""
from __future__ import annotations

import numpy as np

NORMWISE_TOL = 1e-10
COMPONENT_TOL = 1e-8


def parity_metrics(got: np.ndarray, ref: np.ndarray, chunk: int = 4096) -> dict:
    """North-star parity of a whole grid against the oracle's.

    * normwise_max: max over cells of |got - ref| / |ref| (the reference's
      verify metric);
    * floored_componentwise_max: max over components of
      |got - ref| / max(|ref|, 1e-6 |ref_cell|), with the count of components
      above 1e-8 (round 1's definition);
    * floored5_componentwise_max: the same with the floor at 1e-5 |ref_cell|,
      i.e. numpy.allclose(rtol=1e-8, atol=1e-13 |ref_cell|) — the asserted
      component-wise bound: FP64 rounding in two valid orders leaves absolute
      differences of ~1e-15 |ref_cell| on ill-conditioned cells, which a
      1e-6 floor turns into ~1e-8 relative for components near zero;
    * raw_componentwise_max and the count of raw components above 1e-8.
    """
    normwise = floored = floored5 = raw = 0.0
    over = over_floored = comps = 0
    worst = worst_floored = None
    with np.errstate(divide="ignore", invalid="ignore"):
        for a in range(0, got.shape[0], chunk):
            g, r = got[a:a + chunk], ref[a:a + chunk]
            d = np.abs(g - r)
            nrm = np.linalg.norm(r, axis=-1)
            normwise = max(normwise, float((np.linalg.norm(g - r, axis=-1) / nrm).max()))
            fl = d / np.maximum(np.abs(r), 1e-6 * nrm[..., None])
            k = int(np.argmax(fl))
            if fl.flat[k] > floored:
                floored = float(fl.flat[k])
                cell = np.unravel_index(k, fl.shape)
                worst_floored = {"i": int(a + cell[0]), "j": int(cell[1]), "c": int(cell[2]),
                                 "abs_diff": float(d.flat[k]), "abs_ref": float(np.abs(r).flat[k]),
                                 "cell_norm": float(nrm[cell[0], cell[1]])}
            over_floored += int((fl > COMPONENT_TOL).sum())
            floored5 = max(floored5, float((d / np.maximum(np.abs(r), 1e-5 * nrm[..., None])).max()))
            rel = np.where(d == 0, 0.0, d / np.abs(r))
            k = int(np.argmax(rel))
            if rel.flat[k] > raw:
                raw = float(rel.flat[k])
                worst = {"abs_ref": float(np.abs(r).flat[k]),
                         "cell_norm": float(nrm.flat[k // r.shape[-1]])}
            over += int((rel > COMPONENT_TOL).sum())
            comps += rel.size
    return {"cells": int(np.prod(got.shape[:-1])), "components": comps,
            "normwise_max": normwise,
            "floored_componentwise_max": floored, "n_floored_over_1e-8": over_floored,
            "floored_max_at": worst_floored,
            "floored5_componentwise_max": floored5,
            "raw_componentwise_max": raw, "n_raw_over_1e-8": over, "raw_max_at": worst,
            "tolerance": {"normwise": NORMWISE_TOL,
                          "floored5_componentwise (rtol 1e-8, atol 1e-13 |b_cell|)": COMPONENT_TOL},
            "pass": bool(normwise <= NORMWISE_TOL and floored5 <= COMPONENT_TOL),
            "reference": "oracle/ compute_grid (restated gwgrid compute_tile) on the same inputs"}
