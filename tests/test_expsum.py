"""The positive exponential sum behind the genotype grid's low-rank S_BR
(csrc/expsum.cpp): 1/x ~= sum_r w_r exp(-s_r x), checked in extended
precision on the ranges the GLS weights D = 1/(sigma2 (h lambda + 1 - h))
produce.  Host-only."""
import numpy as np
import pytest

from paper_1210_7683_b200.engine import exp_sum_design
from paper_1210_7683_b200.errors import DimensionError


def max_rel_error(s, w, x_min, x_max, points=4001):
    x = np.exp(np.linspace(np.log(x_min), np.log(x_max), points)).astype(np.longdouble)
    x = np.concatenate([x, np.array([x_min, x_max], dtype=np.longdouble)])
    approx = (w.astype(np.longdouble)[None, :] *
              np.exp(-np.outer(x, s.astype(np.longdouble)))).sum(axis=1)
    return float(np.abs(approx * x - 1).max())


@pytest.mark.parametrize("x_min,x_max", [
    (1.0, 1.0), (0.5, 2.0), (0.0889 + 0.0526, 2.883 + 19.0),  # config 1 spectrum, h in [.05,.95]
    (1e-3, 4.0 + 19.0), (1e-6, 1e3), (2.0, 1e9), (1e-9, 1e3)])
def test_relative_accuracy(x_min, x_max):
    s, w = exp_sum_design(x_min, x_max)
    # node 0 (s = 0, w = 0) carries D = 1/sigma2 for h2 = 0; all others positive
    assert len(s) % 64 == 0 and s[0] == 0.0 and w[0] == 0.0
    assert (w[1:] > 0).all() and (np.diff(s) > 0).all()
    assert max_rel_error(s, w, x_min, x_max) < 2.5e-16


def test_terms_grow_logarithmically():
    r = [len(exp_sum_design(1.0, R)[0]) for R in (10.0, 1e3, 1e6, 1e12)]
    assert r == sorted(r) and r[-1] <= 256
    # BASELINE config 1's range (spectrum [0.089, 2.88], h2 in [0.05, 0.95]):
    # 57 terms with the Gauss tail, one 64-column GEMM tile
    assert len(exp_sum_design(0.0889 + 0.0526, 2.883 + 19.0)[0]) == 64


def test_multiple_and_limits():
    s, _ = exp_sum_design(1.0, 100.0, multiple=80)
    assert len(s) % 80 == 0
    with pytest.raises(DimensionError):
        exp_sum_design(0.0, 1.0)
    with pytest.raises(DimensionError):
        exp_sum_design(2.0, 1.0)
    with pytest.raises(DimensionError):
        exp_sum_design(1e-300, 1e300, max_terms=128)


def exp_neg_prod(s, x):
    # split_prep.cuh: exp(-s x) with the product's rounding compensated
    hi = s * x
    lo = (s.astype(np.longdouble) * x - hi).astype(np.float64)  # the fma residual
    return np.exp(-hi) * (1.0 - lo)


def test_factorised_weights_match_direct():
    # D[k, j] from E and F exactly as csrc/split_prep.cuh builds them
    rng = np.random.default_rng(0)
    lam = np.sort(rng.uniform(0.01, 3.0, 300))
    h2 = np.concatenate([rng.uniform(0.05, 0.95, 40), [0.0, 1.0]])
    s2 = rng.uniform(0.5, 2.0, h2.size)
    lam0 = lam.min()
    nz = h2 != 0
    gam = (1 - h2[nz]) / h2[nz]
    s, w = exp_sum_design(lam0 + gam.min(), lam.max() + gam.max())
    e = exp_neg_prod(s[None, :], (lam - lam0)[:, None])
    f = np.zeros((s.size, h2.size))
    for j, (h, v) in enumerate(zip(h2, s2)):
        if h != 0:
            f[:, j] = w * (1 / (v * h)) * exp_neg_prod(s, lam0 + (1 - h) / h)
        else:
            f[0, j] = 1 / v
    # the reference's order (gls.cpp:55-57): sigma2 (h2 lambda + (1 - h2))
    d = 1 / (s2[None, :] * (h2[None, :] * lam[:, None] + (1 - h2[None, :])))
    # sum of r positive terms in double: a few ulps, like D's own rounding
    assert np.abs(e @ f / d - 1).max() < 1.5e-15
