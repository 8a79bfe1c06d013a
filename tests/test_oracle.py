"""The oracle (oracle/gls_oracle.cpp) against the reference's own known-answer
tests and the exact-arithmetic golden vectors.  CPU only.

Each test names the reference test it restates (proj/tests/test_gls.cpp,
test_grid.cpp, acceptance.cpp).  The reference seeds mt19937_64 +
std::normal_distribution, which cannot be reproduced bit-for-bit here, so the
instances are re-drawn with numpy at the same sizes and tolerances.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden.make_golden import load as load_golden


def random_spd(n, rng):
    a = rng.standard_normal((n, n))
    phi = a.T @ a / n + np.eye(n)
    return 0.5 * (phi + phi.T)


def instance(n, p, seed):
    """random_instance (test_gls.cpp:48-63)."""
    rng = np.random.default_rng(seed)
    phi = random_spd(n, rng)
    xl = rng.standard_normal((n, p - 1))
    xr = rng.standard_normal(n)
    y = rng.standard_normal(n)
    return phi, xl, xr, y, float(rng.uniform(0.0, 0.95)), float(rng.uniform(0.25, 4.0))


def rel_err(got, ref):
    return np.linalg.norm(got - ref) / np.linalg.norm(ref)


def test_eigendecomposition_contract():
    """test_gls.cpp:70-97: reconstructs, orthonormal, ascending, signed, repeatable."""
    phi = random_spd(24, np.random.default_rng(7))
    z, lam = orc.eigendecompose(phi)
    assert np.abs(z @ np.diag(lam) @ z.T - phi).max() < 1e-12 * np.abs(phi).max()
    assert np.abs(z.T @ z - np.eye(24)).max() < 1e-13
    assert np.all(np.diff(lam) >= 0)
    at = np.argmax(np.abs(z), axis=0)
    assert np.all(z[at, np.arange(24)] > 0)
    z2, lam2 = orc.eigendecompose(phi)
    assert np.array_equal(z, z2) and np.array_equal(lam, lam2)


def test_eigendecomposition_rejects_asymmetric():
    """test_gls.cpp:99-103."""
    phi = np.eye(5)
    phi[1, 3] = 0.5
    with pytest.raises(orc.OracleError) as e:
        orc.eigendecompose(phi)
    assert orc.CODES[e.value.code] == "non_symmetric"


def test_identity_kinship_flat_spectrum():
    """test_gls.cpp:105-109."""
    _, lam = orc.eigendecompose(np.eye(8))
    assert np.abs(lam - 1.0).max() < 1e-14


def test_trait_weights_formula():
    """test_gls.cpp:111-125."""
    lam = np.array([0.5, 1.0, 2.0, 8.0])
    d, k = orc.trait_weights(lam, 0.25, 3.0)
    ref = 3.0 * (0.25 * lam + 0.75)
    assert np.allclose(d, ref, rtol=1e-15, atol=0)
    assert np.allclose(k, 1 / np.sqrt(ref), rtol=1e-15, atol=0)
    flat, _ = orc.trait_weights(lam, 0.0, 2.0)
    assert np.abs(flat - 2.0).max() == 0.0


def test_nonpositive_weights_rejected_with_coordinates():
    """test_gls.cpp:127-138."""
    with pytest.raises(orc.OracleError) as e:
        orc.trait_weights(np.array([-2.0, 1.0, 4.0]), 0.9, 1.0, trait=17)
    assert e.value.trait_index == 17 and e.value.snp_index == -1


def test_trait_context_quantities():
    """test_gls.cpp:139-157."""
    phi, xl, xr, y, h2, s2 = instance(16, 4, 11)
    z, lam = orc.eigendecompose(phi)
    xl_rot, y_rot = z.T @ xl, z.T @ y
    ctx = orc.trait_context(lam, xl_rot, y_rot, h2, s2, trait=3)
    _, k = orc.trait_weights(lam, h2, s2)
    assert np.abs(ctx["v"] - k * y_rot).max() < 1e-14
    assert np.abs(ctx["w_l"] - k[:, None] * xl_rot).max() < 1e-13
    s_ref = ctx["w_l"].T @ ctx["w_l"]
    assert np.abs(ctx["s_tl"] - s_ref).max() < 1e-12 * np.abs(s_ref).max()
    assert np.abs(ctx["s_tl"] - ctx["s_tl"].T).max() == 0.0
    b_ref = ctx["w_l"].T @ ctx["v"]
    assert np.abs(ctx["b_t"] - b_ref).max() < 1e-12 * (np.abs(b_ref).max() + 1.0)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_partitioned_vs_monolithic(seed):
    """test_gls.cpp:179-191 (<= 1e-13)."""
    phi, xl, xr, y, h2, s2 = instance(32, 4, seed)
    z, lam = orc.eigendecompose(phi)
    mono = orc.solve_single(z, lam, np.column_stack([xl, xr]), y, h2, s2)
    part = orc.solve_partitioned(z, lam, xl, xr, y, h2, s2)
    assert rel_err(part, mono) < 1e-13


@pytest.mark.parametrize("seed", [10, 20, 30, 40])
def test_spectrum_route_vs_cholesky_oracle(seed):
    """test_gls.cpp:193-206 (<= 1e-8)."""
    phi, xl, xr, y, h2, s2 = instance(40, 4, seed)
    z, lam = orc.eigendecompose(phi)
    fast = orc.solve_partitioned(z, lam, xl, xr, y, h2, s2)
    ref = orc.cholesky_solve(phi, np.column_stack([xl, xr]), y, h2, s2)
    assert rel_err(fast, ref) < 1e-8


def test_spectral_inverse():
    """test_gls.cpp:208-217."""
    phi, *_ , h2, s2 = instance(24, 3, 77)
    z, lam = orc.eigendecompose(phi)
    d, _ = orc.trait_weights(lam, h2, s2)
    m_inv = z @ np.diag(1 / d) @ z.T
    m = s2 * (h2 * phi + (1 - h2) * np.eye(24))
    assert np.abs(m @ m_inv - np.eye(24)).max() < 1e-8


@pytest.mark.parametrize("scale", [0.125, 1.0, 64.0])
def test_sigma2_invariance(scale):
    """test_gls.cpp:219-232 (<= 1e-12)."""
    phi, xl, xr, y, h2, s2 = instance(28, 4, 99)
    z, lam = orc.eigendecompose(phi)
    b0 = orc.solve_partitioned(z, lam, xl, xr, y, h2, s2)
    b1 = orc.solve_partitioned(z, lam, xl, xr, y, h2, s2 * scale)
    assert rel_err(b1, b0) < 1e-12


def test_residual_orthogonality():
    """test_gls.cpp:234-247."""
    phi, xl, xr, y, h2, s2 = instance(36, 5, 123)
    z, lam = orc.eigendecompose(phi)
    x = np.column_stack([xl, xr])
    b = orc.solve_partitioned(z, lam, xl, xr, y, h2, s2)
    m = s2 * (h2 * phi + (1 - h2) * np.eye(36))
    grad = x.T @ np.linalg.solve(m, y - x @ b)
    rhs = x.T @ np.linalg.solve(m, y)
    assert np.abs(grad).max() < 1e-8 * (np.abs(rhs).max() + 1.0)


def test_identity_kinship_cholesky_is_ols():
    """test_gls.cpp:249-260."""
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal((30, 3)), rng.standard_normal(30)
    b = orc.cholesky_solve(np.eye(30), x, y, 0.6, 2.5)
    ols = np.linalg.solve(x.T @ x, x.T @ y)
    assert rel_err(b, ols) < 1e-12


def test_single_predictor_without_covariates():
    """test_gls.cpp:262-272 (p = 1)."""
    phi, _, xr, y, h2, s2 = instance(16, 2, 31)
    z, lam = orc.eigendecompose(phi)
    part = orc.solve_partitioned(z, lam, np.zeros((16, 0)), xr, y, h2, s2)
    ref = orc.cholesky_solve(phi, xr, y, h2, s2)
    assert part.shape == (1,) and rel_err(part, ref) < 1e-8


def test_zero_variant_column_npd_with_coordinates():
    """test_gls.cpp:274-292 and test_grid.cpp:689-730: a zero variant column
    fails positive definiteness; the serial traversal reports the first bad
    cell in grid order."""
    phi, xl, _, _, _, _ = instance(12, 3, 47)
    rng = np.random.default_rng(47)
    z, lam = orc.eigendecompose(phi)
    snps = rng.standard_normal((12, 43))
    snps[:, 42] = 0.0
    traits = rng.standard_normal((12, 7))
    h2, s2 = np.full(7, 0.5), np.ones(7)
    with pytest.raises(orc.OracleError) as e:
        orc.compute_grid(lam, z.T @ xl, z.T @ snps, z.T @ traits, h2, s2, workers=1)
    assert (e.value.snp_index, e.value.trait_index) == (42, 0)
    with pytest.raises(orc.OracleError) as e:
        orc.compute_grid(lam, z.T @ xl, z.T @ snps, z.T @ traits, h2, s2, workers=4)
    assert e.value.snp_index == 42 and 0 <= e.value.trait_index < 7


def test_h2_zero_is_ols():
    """test_gls.cpp:294-306 (<= 1e-10)."""
    phi, xl, xr, y, _, _ = instance(20, 4, 61)
    z, lam = orc.eigendecompose(phi)
    fast = orc.solve_partitioned(z, lam, xl, xr, y, 0.0, 1.5)
    x = np.column_stack([xl, xr])
    assert rel_err(fast, np.linalg.solve(x.T @ x, x.T @ y)) < 1e-10


def test_trait_weight_failure_surfaces_trait_index():
    """test_grid.cpp:732-773: an indefinite kinship with high heritability
    fails at context build with (snp -1, trait j)."""
    n = 8
    lam = np.arange(n) - 0.5
    rng = np.random.default_rng(3)
    h2 = np.zeros(5)
    h2[3] = 0.9
    with pytest.raises(orc.OracleError) as e:
        orc.compute_grid(lam, np.ones((n, 1)), rng.standard_normal((n, 4)),
                         rng.standard_normal((n, 5)), h2, np.ones(5))
    assert (e.value.snp_index, e.value.trait_index) == (-1, 3)


def test_grid_block_and_worker_invariance():
    """test_grid.cpp:286-336 / acceptance criterion 4: bitwise identical for
    any block shape and worker count."""
    rng = np.random.default_rng(2)
    n, m, t = 48, 37, 11
    phi = random_spd(n, rng)
    z, lam = orc.eigendecompose(phi)
    xl = np.column_stack([np.ones(n), rng.standard_normal((n, 2))])
    snps = rng.integers(0, 3, (n, m)).astype(float)
    traits = rng.standard_normal((n, t))
    h2, s2 = rng.uniform(0.05, 0.95, t), np.ones(t)
    args = (lam, z.T @ xl, z.T @ snps, z.T @ traits, h2, s2)
    base = orc.compute_grid(*args, workers=1)
    for workers, mbb, tbb in ((4, 0, 0), (3, 5, 2), (2, 1, 1), (8, 37, 11)):
        assert np.array_equal(base, orc.compute_grid(*args, workers=workers, mbb=mbb, tbb=tbb))
    stream = orc.compute_grid(*args, layout="stream")
    assert np.array_equal(stream.transpose(1, 0, 2), base)


def test_acceptance_criterion_1():
    """acceptance.cpp:110-163: n=64, p=4, m=100, t=50, 5000 cells vs the
    Cholesky oracle <= 1e-8 (recorded 2.638e-14, test_output.txt:19)."""
    from paper_1210_7683_b200 import datagen

    ds = datagen.generate(64, 4, 100, 50, seed=20260816)
    b = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                       ds["sigma2"], workers=4)
    ii, jj = np.meshgrid(np.arange(100), np.arange(50), indexing="ij")
    ref = orc.cholesky_cells(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                             ds["sigma2"], ii.ravel(), jj.ravel())
    rel = np.linalg.norm(b.reshape(-1, 4) - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-8
    assert rel.max() < 1e-12  # the restatement is as accurate as the reference's 2.6e-14


def test_oracle_against_exact_rotated_goldens():
    """The cell math against exact-arithmetic answers (tests/golden/rotated.json)."""
    for case in load_golden("rotated.json"):
        n, p, m, t = case["n"], case["p"], case["m"], case["t"]
        args = (case["lambda"], case["xl_rot"], case["snps_rot"], case["traits_rot"],
                case["h2"], case["sigma2"])
        if case["ok"].all():
            b = orc.compute_grid(*args)
            rel = np.linalg.norm(b - case["b"], axis=2) / np.linalg.norm(case["b"], axis=2)
            assert rel.max() < 1e-13, (n, p, rel.max())
        else:
            with pytest.raises(orc.OracleError) as e:
                orc.compute_grid(*args)
            bad = np.argwhere(~case["ok"])
            first = min((int(j), int(i)) for i, j in bad)
            assert (e.value.trait_index, e.value.snp_index) == first


def test_oracle_against_exact_dense_goldens():
    """Whole chain (eig + rotation + cell) against exact GLS answers."""
    for case in load_golden("dense.json"):
        b = orc.solve_grid(case["kinship"], case["xl"], case["snps"], case["traits"],
                           case["h2"], case["sigma2"])
        rel = np.linalg.norm(b - case["b"], axis=2) / np.linalg.norm(case["b"], axis=2)
        assert rel.max() < 1e-11, rel.max()
