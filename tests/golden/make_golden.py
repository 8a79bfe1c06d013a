"""Generate exact-arithmetic golden vectors for the GLS cell (committed fixtures).

The reference ships no golden b vectors, so these fixtures pin
both the oracle and the device kernel to the *exact* solution of each tiny GLS
problem, computed with Python `fractions` from the double-precision inputs
(every double is an exact rational), then rounded once to double.

Two families:
* rotated.json — operands already in the eigenbasis (lambda, X_L', x', y'),
  exact b = (X'^T D X')^-1 X'^T D y', D = diag(1 / (sigma2 (h2 lambda + 1 - h2))):
  pins build_trait_context + solve_gls_cell (gls.cpp:48-132) with no
  eigendecomposition involved (run with basis = I).
* dense.json — raw operands with a dense SPD kinship Phi, exact
  b = (X^T M^-1 X)^-1 X^T M^-1 y, M = sigma2 (h2 Phi + (1 - h2) I): pins the
  whole chain (eigendecomposition + rotation + cell) like the reference's
  Cholesky oracle (gls.cpp:188-244) does, but exactly.
Edge cases: p = 1, h2 = 0 (OLS), a zero variant column (expected NPD).

Run: python tests/golden/make_golden.py   (rewrites the two JSON files)
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def F(x: float) -> Fraction:
    return Fraction(float(x))


def solve_exact(a: list[list[Fraction]], b: list[Fraction]) -> list[Fraction] | None:
    """Gaussian elimination with partial pivoting in exact arithmetic."""
    n = len(b)
    m = [row[:] + [b[i]] for i, row in enumerate(a)]
    for c in range(n):
        piv = next((r for r in range(c, n) if m[r][c] != 0), None)
        if piv is None:
            return None
        m[c], m[piv] = m[piv], m[c]
        for r in range(n):
            if r != c and m[r][c] != 0:
                f = m[r][c] / m[c][c]
                m[r] = [x - f * y for x, y in zip(m[r], m[c])]
    return [m[i][n] / m[i][i] for i in range(n)]


def gls_exact(x_cols: list[list[Fraction]], y: list[Fraction], minv_apply) -> list[float] | None:
    """b = (X^T W X)^-1 X^T W y with W applied by minv_apply(v) -> W v."""
    wx = [minv_apply(c) for c in x_cols]
    wy = minv_apply(y)
    p = len(x_cols)
    s = [[sum(xi * wj for xi, wj in zip(x_cols[a], wx[b])) for b in range(p)] for a in range(p)]
    r = [sum(xi * wi for xi, wi in zip(x_cols[a], wy)) for a in range(p)]
    # positive definiteness of the normal matrix (exact): all leading minors > 0
    sol = solve_exact(s, r)
    if sol is None:
        return None
    for k in range(1, p + 1):
        sub = [row[:k] for row in s[:k]]
        det = _det(sub)
        if det <= 0:
            return None
    return [float(v) for v in sol]


def _det(a: list[list[Fraction]]) -> Fraction:
    n = len(a)
    m = [row[:] for row in a]
    det = Fraction(1)
    for c in range(n):
        piv = next((r for r in range(c, n) if m[r][c] != 0), None)
        if piv is None:
            return Fraction(0)
        if piv != c:
            m[c], m[piv] = m[piv], m[c]
            det = -det
        det *= m[c][c]
        for r in range(c + 1, n):
            f = m[r][c] / m[c][c]
            m[r] = [x - f * y for x, y in zip(m[r], m[c])]
    return det


def hexs(a) -> list:
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel(order="F")]


def rotated_case(rng, n, p, m, t, zero_col=None, h2_zero=False):
    lam = np.sort(rng.uniform(0.05, 3.0, n))
    xl = rng.standard_normal((n, p - 1))
    xr = rng.integers(0, 3, (n, m)).astype(np.float64) + rng.standard_normal((n, m)) * 0.25
    if zero_col is not None:
        xr[:, zero_col] = 0.0
    y = rng.standard_normal((n, t))
    h2 = rng.uniform(0.05, 0.95, t)
    if h2_zero:
        h2[0] = 0.0
    sigma2 = rng.uniform(0.5, 2.0, t)
    b = []
    for j in range(t):
        d = [F(sigma2[j]) * (F(h2[j]) * F(lam[k]) + (1 - F(h2[j]))) for k in range(n)]
        apply = lambda v, d=d: [vi / di for vi, di in zip(v, d)]  # noqa: E731
        col = []
        for i in range(m):
            xs = [[F(v) for v in xl[:, c]] for c in range(p - 1)] + [[F(v) for v in xr[:, i]]]
            col.append(gls_exact(xs, [F(v) for v in y[:, j]], apply))
        b.append(col)
    return {
        "n": n, "p": p, "m": m, "t": t,
        "lambda": hexs(lam), "xl_rot": hexs(xl), "snps_rot": hexs(xr), "traits_rot": hexs(y),
        "h2": hexs(h2), "sigma2": hexs(sigma2),
        # b[j][i] = list of p floats (hex) or null when the cell is not PD
        "b": [[None if c is None else [v.hex() for v in c] for c in col] for col in b],
    }


def dense_case(rng, n, p, m, t):
    a = rng.standard_normal((n, n))
    phi = a @ a.T / n + np.eye(n)
    phi = 0.5 * (phi + phi.T)
    xl = np.column_stack([np.ones(n), rng.standard_normal((n, p - 2))]) if p >= 2 else np.zeros((n, 0))
    xr = rng.integers(0, 3, (n, m)).astype(np.float64)
    y = rng.standard_normal((n, t))
    h2 = rng.uniform(0.05, 0.95, t)
    sigma2 = np.ones(t)
    phiF = [[F(phi[r, c]) for c in range(n)] for r in range(n)]
    b = []
    for j in range(t):
        mm = [[F(sigma2[j]) * (F(h2[j]) * phiF[r][c] + ((1 - F(h2[j])) if r == c else 0))
               for c in range(n)] for r in range(n)]
        apply = lambda v, mm=mm: solve_exact(mm, v)  # noqa: E731
        col = []
        for i in range(m):
            xs = [[F(v) for v in xl[:, c]] for c in range(p - 1)] + [[F(v) for v in xr[:, i]]]
            col.append(gls_exact(xs, [F(v) for v in y[:, j]], apply))
        b.append(col)
    return {
        "n": n, "p": p, "m": m, "t": t,
        "kinship": hexs(phi), "xl": hexs(xl), "snps": hexs(xr), "traits": hexs(y),
        "h2": hexs(h2), "sigma2": hexs(sigma2),
        "b": [[None if c is None else [v.hex() for v in c] for c in col] for col in b],
    }


def main():
    rng = np.random.default_rng(1210_7683)
    rotated = [
        rotated_case(rng, 6, 1, 3, 2),
        rotated_case(rng, 8, 2, 4, 3),
        rotated_case(rng, 9, 3, 4, 2, h2_zero=True),
        rotated_case(rng, 12, 4, 5, 3),
        rotated_case(rng, 10, 4, 3, 2, zero_col=1),
        rotated_case(rng, 11, 5, 3, 2),
    ]
    dense = [
        dense_case(rng, 6, 2, 3, 2),
        dense_case(rng, 8, 3, 3, 2),
        dense_case(rng, 10, 4, 4, 2),
    ]
    with open(os.path.join(HERE, "rotated.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "cases": rotated}, f)
    with open(os.path.join(HERE, "dense.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "cases": dense}, f)


def load(name: str) -> list[dict]:
    """Decode a fixture file into numpy arrays (tests use this)."""
    with open(os.path.join(HERE, name)) as f:
        raw = json.load(f)["cases"]
    out = []
    for c in raw:
        n, p, m, t = c["n"], c["p"], c["m"], c["t"]
        dec = {"n": n, "p": p, "m": m, "t": t}
        for key, val in c.items():
            if key in ("n", "p", "m", "t", "b"):
                continue
            arr = np.array([float.fromhex(v) for v in val])
            shape = {"lambda": (n,), "h2": (t,), "sigma2": (t,), "kinship": (n, n),
                     "xl_rot": (n, p - 1), "xl": (n, p - 1), "snps_rot": (n, m), "snps": (n, m),
                     "traits_rot": (n, t), "traits": (n, t)}[key]
            dec[key] = np.asfortranarray(arr.reshape(shape, order="F"))
        b = np.full((m, t, p), np.nan)
        ok = np.ones((m, t), dtype=bool)
        for j, col in enumerate(c["b"]):
            for i, cell in enumerate(col):
                if cell is None:
                    ok[i, j] = False
                else:
                    b[i, j] = [float.fromhex(v) for v in cell]
        dec["b"] = b
        dec["ok"] = ok
        out.append(dec)
    return out


if __name__ == "__main__":
    main()
