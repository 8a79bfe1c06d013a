"""Randomised parity sweeps.

CPU: the oracle against exact rational arithmetic on random tiny problems
(hypothesis-driven), pinning the restatement beyond the fixed golden files.
GPU: the device grid against the oracle over a seeded sweep of shapes,
including the degenerate edges the reference allows (m = 1, t = 1, p = 1,
n = p, n not a multiple of the k tile, t not a multiple of the trait tile).
"""
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as orc
from tests.golden.make_golden import gls_exact


def exact_cells(lam, xl, xr, y, h2, s2):
    F = Fraction
    d = [F(s2) * (F(h2) * F(v) + (1 - F(h2))) for v in lam]
    apply = lambda v: [a / b for a, b in zip(v, d)]  # noqa: E731
    out = []
    for i in range(xr.shape[1]):
        cols = [[F(v) for v in xl[:, c]] for c in range(xl.shape[1])] + [[F(v) for v in xr[:, i]]]
        out.append(gls_exact(cols, [F(v) for v in y], apply))
    return out


@settings(max_examples=40, deadline=None, derandomize=True)
@given(n=st.integers(2, 9), pm1=st.integers(0, 3), m=st.integers(1, 3),
       seed=st.integers(0, 2**32 - 1), h2=st.floats(0.0, 0.95), s2=st.floats(0.25, 4.0))
def test_oracle_cells_match_exact_arithmetic(n, pm1, m, seed, h2, s2):
    if pm1 + 1 > n:
        return
    rng = np.random.default_rng(seed)
    lam = np.sort(rng.uniform(0.05, 3.0, n))
    xl = rng.standard_normal((n, pm1))
    xr = rng.standard_normal((n, m))
    y = rng.standard_normal((n, 1))
    exact = exact_cells(lam, xl, xr, y[:, 0], h2, s2)
    if any(e is None for e in exact):
        return
    got = orc.compute_grid(lam, xl, xr, y, [h2], [s2])[:, 0, :]
    ref = np.array(exact)
    # relative to the cell norm, scaled by the conditioning of the weighted
    # tiny system (the normal equations square it); small constant for the
    # O(n p) rounding steps of the context + cell
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    w = 1.0 / np.sqrt(s2 * (h2 * lam + (1.0 - h2)))
    cond = max(np.linalg.cond(w[:, None] * np.column_stack([xl, xr[:, i]])) for i in range(m))
    assert rel.max() <= 8e-14 * max(1.0, cond) ** 2


def _shapes():
    rng = np.random.default_rng(1210)
    out = [(1, 1, 1, 1), (2, 2, 3, 2), (5, 5, 4, 3), (33, 4, 1, 1), (64, 4, 1, 33),
           (65, 3, 129, 1), (96, 12, 17, 16), (129, 24, 9, 9)]
    while len(out) < 30:
        n = int(rng.integers(8, 700))
        p = int(rng.integers(1, min(24, n - 3) + 1))
        out.append((n, p, int(rng.integers(1, 400)), int(rng.integers(1, 80))))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,m,t", _shapes())
def test_device_sweep_matches_oracle(n, p, m, t):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1210_7683_b200 as gw
    from paper_1210_7683_b200 import datagen

    ds = datagen.generate(n, p, m, t, seed=n * 7 + p)
    basis, values = gw.eigendecompose(ds["kinship"])
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        try:
            got = eng.run_grid(ds["snps"])
        except gw.NotPositiveDefiniteError as e:
            # tiny n = p systems can be singular; the oracle must agree
            with pytest.raises(orc.OracleError) as oe:
                orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                                 orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"])
            assert (oe.value.snp_index, oe.value.trait_index) == (e.snp_index, e.trait_index)
            return
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                           orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)
    assert not np.isnan(got).any()
    nrm = np.linalg.norm(ref, axis=2)
    normwise = np.linalg.norm(got - ref, axis=2) / nrm
    # The reference's acceptance bound is 1e-8 (acceptance.cpp:110-163).  Both
    # routes are backward stable; what is left is cancellation in the n-term
    # sums (visible at p = 1, where the cell norm is one dot-product ratio)
    # and, for n close to p, the conditioning of the p x p systems.
    tol = 1e-10 if n >= p + 4 else 1e-9
    assert normwise.max() <= tol, (normwise.max(), n, p)
    floored = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-6 * nrm[..., None])
    assert floored.max() <= 1e-8, (floored.max(), n, p)
