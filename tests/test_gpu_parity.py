"""Device parity: the CUDA path (through the C ABI) against the oracle and the
exact-arithmetic golden vectors.  Needs a B200.

Tolerances (BASELINE.json north star: b_ij within 1e-8 max component-wise
relative error of the CPU oracle):
  * norm-wise per cell (the reference's own verify metric,
    gwgrid_main.cpp:378-380):             <= 1e-10 (100x under the
    reference's own 1e-8 acceptance bound; p = 1 cells are a single
    dot-product ratio, so cancellation in the n-term sums shows up to ~1e-11)
  * component-wise, floored at 1e-6 of the cell norm (components whose exact
    value is ~0 have no meaningful relative error for ANY two rounding
    orders):                <= 1e-8
  * raw component-wise is reported, and asserted <= 1e-8 on components with
    |b| >= 1e-3 |b_cell|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1210_7683_b200 as gw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402
from tests.golden.make_golden import load as load_golden  # noqa: E402

NORMWISE = 1e-10
COMPONENT = 1e-8


def metrics(got, ref):
    nrm = np.linalg.norm(ref, axis=-1, keepdims=True)
    diff = np.abs(got - ref)
    normwise = (np.linalg.norm(got - ref, axis=-1) / nrm[..., 0]).max()
    floored = (diff / np.maximum(np.abs(ref), 1e-6 * nrm)).max()
    big = np.abs(ref) >= 1e-3 * nrm
    raw_big = (diff[big] / np.abs(ref[big])).max() if big.any() else 0.0
    raw = (diff / np.abs(ref)).max()
    return normwise, floored, raw_big, raw


def assert_parity(got, ref):
    assert not np.isnan(got).any()
    normwise, floored, raw_big, raw = metrics(got, ref)
    assert normwise <= NORMWISE, f"norm-wise {normwise:.3e} (raw component-wise {raw:.3e})"
    assert floored <= COMPONENT, f"floored component-wise {floored:.3e}"
    assert raw_big <= COMPONENT, f"component-wise on |b|>=1e-3|b| {raw_big:.3e}"


def oracle_grid(ds, basis, values):
    return orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                            orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)


def device_grid(ds, basis, values, **kw):
    n, p = ds["kinship"].shape[0], ds["xl"].shape[1] + 1
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        return eng.run_grid(ds["snps"], **kw)


@pytest.mark.parametrize("n,p,m,t", [
    (1000, 4, 4000, 100),    # config 0 shape (m reduced)
    (257, 4, 333, 37),       # ragged everything
    (64, 1, 50, 9),          # p = 1: no covariates
    (96, 2, 70, 17),
    (130, 3, 65, 40),
    (200, 5, 150, 33),
    (300, 7, 130, 21),
    (320, 12, 80, 19),
    (500, 20, 70, 13),       # config 4's p
    (31, 24, 20, 5),         # n < 32
    (40, 32, 20, 5),         # largest compiled p
])
def test_grid_matches_oracle(n, p, m, t):
    ds = datagen.generate(n, p, m, t, seed=n + p)
    basis, values = gw.eigendecompose(ds["kinship"])
    got = device_grid(ds, basis, values)
    ref = oracle_grid(ds, basis, values)
    assert_parity(got, ref)


def test_rotated_golden_vectors_exact():
    """Exact-arithmetic cells (tests/golden/rotated.json), basis = I."""
    for case in load_golden("rotated.json"):
        n, p, m, t = case["n"], case["p"], case["m"], case["t"]
        with gw.Engine(n, p) as eng:
            eng.set_spectrum(np.eye(n), case["lambda"])
            eng.set_covariates(case["xl_rot"])
            eng.set_traits(case["traits_rot"], case["h2"], case["sigma2"], rotated=True)
            if case["ok"].all():
                got = eng.solve_snp_slab(case["snps_rot"], rotated=True)
                rel = np.linalg.norm(got - case["b"], axis=2) / np.linalg.norm(case["b"], axis=2)
                assert rel.max() < 1e-13, (n, p, rel.max())
            else:
                with pytest.raises(gw.NotPositiveDefiniteError) as e:
                    eng.solve_snp_slab(case["snps_rot"], rotated=True)
                bad = np.argwhere(~case["ok"])
                first = min((int(j), int(i)) for i, j in bad)
                assert (e.value.trait_index, e.value.snp_index) == first


def test_dense_golden_vectors_exact():
    for case in load_golden("dense.json"):
        res = gw.solve_grid(case["kinship"], case["xl"], case["snps"], case["traits"],
                            case["h2"], case["sigma2"])
        rel = np.linalg.norm(res["b"] - case["b"], axis=2) / np.linalg.norm(case["b"], axis=2)
        assert rel.max() < 1e-11, rel.max()


def test_full_pipeline_matches_oracle_solve_grid():
    """gwgrid.solve_grid contract end to end (eig on CPU, everything else on
    the device) vs the oracle's in-core restatement of solve_grid."""
    ds = datagen.generate(256, 4, 300, 40, seed=7)
    res = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                        ds["sigma2"])
    ref = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                         ds["sigma2"], workers=8)
    assert res["b"].shape == (300, 40, 4)
    assert_parity(res["b"], ref)
    c = res["counters"]
    assert c["kernel_launches"] >= 3 and c["loop_flops"] > 0 and c["loop_transform_flops"] == 0
    assert c["bytes_stored"] == 300 * 40 * 4 * 8


def test_cholesky_oracle_spot_checks():
    """acceptance.cpp criterion 1 on the device: cells vs the independent
    Cholesky route (dense M, no eigendecomposition)."""
    ds = datagen.generate(64, 4, 100, 50, seed=20260816)
    res = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                        ds["sigma2"])
    ii, jj = np.meshgrid(np.arange(100), np.arange(50), indexing="ij")
    ref = orc.cholesky_cells(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                             ds["sigma2"], ii.ravel(), jj.ravel())
    got = res["b"].reshape(-1, 4)
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-8  # the reference's acceptance bound
    assert rel.max() < 1e-12


def test_bitwise_invariance_across_slabs_layouts_and_entry_points():
    """The reference guarantees byte-identical output for any tiling
    (grid.hpp:35-38); here: any slab width, buffering, layout, entry point
    and host/device placement."""
    ds = datagen.generate(300, 4, 1000, 70, seed=3)
    basis, values = gw.eigendecompose(ds["kinship"])
    base = device_grid(ds, basis, values)
    for mb in (1, 7, 128, 333, 999):
        assert np.array_equal(base, device_grid(ds, basis, values, mb=mb))
    assert np.array_equal(base, device_grid(ds, basis, values, mb=100, double_buffer=False))
    stream = device_grid(ds, basis, values, layout="stream", mb=256)
    assert np.array_equal(stream.transpose(1, 0, 2), base)
    with gw.Engine(300, 4) as eng:
        eng.set_spectrum(torch.from_numpy(basis).cuda(), torch.from_numpy(values).cuda())
        eng.set_covariates(torch.from_numpy(np.asarray(ds["xl"])).cuda())
        eng.set_traits(torch.from_numpy(np.asarray(ds["traits"])).cuda(),
                       torch.from_numpy(ds["h2"]).cuda(), torch.from_numpy(ds["sigma2"]).cuda())
        xd = torch.from_numpy(np.asarray(ds["snps"])).cuda()
        out = torch.empty((1000, 70, 4), dtype=torch.float64, device="cuda")
        eng.solve_snp_slab(xd, out=out)
        assert np.array_equal(out.cpu().numpy(), base)
        # slab-by-slab through solve_snp_slab with global offsets
        parts = [eng.solve_snp_slab(np.asfortranarray(ds["snps"][:, a:b]), i0=a)
                 for a, b in ((0, 1), (1, 500), (500, 1000))]
        assert np.array_equal(np.concatenate(parts, axis=0), base)


CODINGS = pytest.mark.parametrize("coding", ["real", "genotypes"])


@CODINGS
def test_zero_snp_column_fails_with_coordinates(coding):
    """test_gls.cpp:274-292 / test_grid.cpp:689-730 on the device."""
    ds = datagen.generate(48, 3, 12, 6, seed=4)
    snps = ds["snps"].copy()
    snps[:, 5] = 0.0
    with pytest.raises(gw.NotPositiveDefiniteError, match="positive definite") as e:
        gw.solve_grid(ds["kinship"], ds["xl"], snps, ds["traits"], ds["h2"], ds["sigma2"],
                      snp_coding=coding)
    assert (e.value.snp_index, e.value.trait_index) == (5, 0)
    with pytest.raises(ValueError):  # reference's Python mapping
        gw.solve_grid(ds["kinship"], ds["xl"], snps, ds["traits"], ds["h2"], ds["sigma2"], mb=5,
                      snp_coding=coding)


@CODINGS
def test_trait_weight_failure_reports_trait(coding):
    """test_grid.cpp:732-773: indefinite kinship + high h2 -> (-1, j)."""
    n = 8
    phi = np.diag(np.arange(n) - 0.5)
    rng = np.random.default_rng(3)
    h2 = np.zeros(5)
    h2[3] = 0.9
    with pytest.raises(gw.NotPositiveDefiniteError) as e:
        gw.solve_grid(phi, np.ones((n, 1)), rng.integers(0, 3, (n, 4)).astype(float),
                      rng.standard_normal((n, 5)), h2, np.ones(5), snp_coding=coding)
    assert (e.value.snp_index, e.value.trait_index) == (-1, 3)


@CODINGS
def test_singular_covariates_fail_every_cell_of_the_trait(coding):
    """S_TL singular (a zero covariate column): the reference's full LLT fails
    at the first cell of the trait; the device reports (first SNP, first
    trait)."""
    ds = datagen.generate(40, 4, 9, 3, seed=8)
    xl = ds["xl"].copy()
    xl[:, 2] = 0.0
    with pytest.raises(gw.NotPositiveDefiniteError) as e:
        gw.solve_grid(ds["kinship"], xl, ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                      snp_coding=coding)
    assert (e.value.snp_index, e.value.trait_index) == (0, 0)


@CODINGS
def test_h2_zero_is_ols_and_sigma2_invariance(coding):
    ds = datagen.generate(60, 4, 20, 6, seed=12)
    x_all = ds["xl"]
    h2 = np.zeros(6)
    b = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], h2, np.ones(6),
                      snp_coding=coding)["b"]
    for i in (0, 7, 19):
        x = np.column_stack([x_all, ds["snps"][:, i]])
        ols = np.linalg.lstsq(x, ds["traits"], rcond=None)[0].T
        rel = np.linalg.norm(b[i] - ols, axis=1) / np.linalg.norm(ols, axis=1)
        assert rel.max() < 1e-10
    b1 = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                       np.ones(6), snp_coding=coding)["b"]
    b2 = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                       np.full(6, 64.0), snp_coding=coding)["b"]
    assert (np.linalg.norm(b1 - b2, axis=2) / np.linalg.norm(b1, axis=2)).max() < 1e-12


def test_solve_cell_matches_partitioned_oracle():
    ds = datagen.generate(50, 3, 4, 3, seed=2)
    z, lam = gw.eigendecompose(ds["kinship"])
    got = gw.solve_cell(ds["kinship"], ds["xl"], ds["snps"][:, 2], ds["traits"][:, 1],
                        float(ds["h2"][1]), 1.0)
    ref = orc.solve_partitioned(z, lam, ds["xl"], ds["snps"][:, 2], ds["traits"][:, 1],
                                float(ds["h2"][1]), 1.0)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


@CODINGS
def test_config1_full_size_properties(coding):
    """BASELINE configs[1] at full size (n=1000, p=4, m=1e5, t=1e3), both SNP
    codings (genotypes = the bench path): size-independent properties — no
    NaN, bitwise-equal results for two slab widths (checksum of checksums),
    and seeded random spot checks against the oracle and the Cholesky route."""
    n, p, m, t = 1000, 4, 100_000, 1000
    ds = datagen.generate(n, p, m, t, seed=1)
    basis, values = gw.eigendecompose(ds["kinship"])
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        b = eng.run_grid(ds["snps"])
        b2 = eng.run_grid(ds["snps"], mb=4736)
    assert not np.isnan(b).any()
    assert np.array_equal(b.view(np.uint64).sum(axis=(1, 2)), b2.view(np.uint64).sum(axis=(1, 2)))
    rng = np.random.default_rng(99)
    ii = rng.integers(0, m, 64)
    jj = rng.integers(0, t, 64)
    cols = np.unique(ii)
    sub = {k: ds[k] for k in ("kinship", "xl", "traits", "h2", "sigma2")}
    sub["snps"] = np.asfortranarray(ds["snps"][:, cols])
    ref = oracle_grid(sub, basis, values)
    pos = {c: k for k, c in enumerate(cols)}
    got = np.stack([b[i, j] for i, j in zip(ii, jj)])
    want = np.stack([ref[pos[i], j] for i, j in zip(ii, jj)])
    assert_parity(got, want)
    chol = orc.cholesky_cells(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                              ds["sigma2"], ii[:8], jj[:8])
    rel = np.linalg.norm(got[:8] - chol, axis=1) / np.linalg.norm(chol, axis=1)
    assert rel.max() < 1e-10


def test_device_eigendecomposition_contract():
    """gwg_eigendecompose keeps eigendecompose_kinship's contract
    (gls.cpp:16-46; test_gls.cpp:70-109)."""
    ds = datagen.generate(300, 3, 2, 2, seed=21)
    phi = ds["kinship"]
    z, lam = gw.eigendecompose(phi, device=0)
    assert np.all(np.diff(lam) >= 0)
    assert np.abs(z @ np.diag(lam) @ z.T - phi).max() < 1e-12 * np.abs(phi).max() * 10
    assert np.abs(z.T @ z - np.eye(300)).max() < 1e-12
    at = np.argmax(np.abs(z), axis=0)
    assert np.all(z[at, np.arange(300)] > 0)
    zc, lc = gw.eigendecompose(phi)
    assert np.abs(lam - lc).max() < 1e-12 * np.abs(lc).max()
    bad = np.eye(5)
    bad[1, 3] = 0.5
    with pytest.raises(gw.NonSymmetricError):
        gw.eigendecompose(bad, device=0)
    _, flat = gw.eigendecompose(np.eye(8), device=0)
    assert np.abs(flat - 1.0).max() < 1e-14


def test_device_eig_full_chain_matches_oracle():
    """solve_grid with the eigendecomposition on the device: b is invariant to
    the choice of eigenbasis, so it still matches the oracle's CPU chain."""
    ds = datagen.generate(400, 4, 200, 30, seed=17)
    res = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                        ds["sigma2"], device_eig=True)
    ref = orc.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                         ds["sigma2"], workers=8)
    normwise, floored, _, _ = metrics(res["b"], ref)
    assert normwise < 1e-10 and floored < 1e-8


def test_device_verify_grid_matches_reference_contract():
    """gwgrid.verify_grid (bindings.cpp:192-222) on the device: the Cholesky
    route accepts the engine's grid and flags a corrupted cell
    (test_cli.cpp:199-226)."""
    ds = datagen.generate(200, 4, 150, 20, seed=31)
    args = (ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    b = gw.solve_grid(*args)["b"]
    err = gw.verify_grid(*args, b)
    assert err < 1e-11
    # agrees with the oracle's Cholesky route on a few cells
    ref = orc.cholesky_cells(*args, [0, 77, 149], [0, 5, 19])
    got = np.stack([b[0, 0], b[77, 5], b[149, 19]])
    assert (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max() < 1e-11
    bad = b.copy()
    bad[77, 5, 2] += 1e-3 * np.abs(bad[77, 5]).max()
    assert gw.verify_grid(*args, bad) > 1e-5
    # p = 1
    b1 = gw.solve_grid(ds["kinship"], np.zeros((200, 0)), ds["snps"], ds["traits"], ds["h2"],
                       ds["sigma2"])["b"]
    assert gw.verify_grid(ds["kinship"], np.zeros((200, 0)), ds["snps"], ds["traits"], ds["h2"],
                          ds["sigma2"], b1) < 1e-11


def test_engine_argument_errors():
    """The C ABI rejects empty / mismatched operands with DimensionError."""
    with gw.Engine(16, 3) as eng:
        with pytest.raises(gw.DimensionError, match="set_traits"):
            eng.solve_snp_slab(np.ones((16, 2)))
        eng.set_spectrum(np.eye(16), np.ones(16))
        eng.set_covariates(np.ones((16, 2)))
        with pytest.raises(gw.DimensionError):
            eng.set_traits(np.ones((16, 0)), [], [])
        eng.set_traits(np.ones((16, 2)), [0.5, 0.5], [1.0, 1.0])
        with pytest.raises(gw.DimensionError):
            eng.solve_snp_slab(np.ones((15, 2)))
        with pytest.raises(gw.DimensionError):
            eng.run_grid(np.ones((16, 0)))


def test_subnormal_pivot_is_solved_not_flushed():
    """A positive but subnormal Schur pivot (x nearly in the span of X_L, all
    scaled by 1e-150) is a valid cell for the reference's LLT; the device's
    reciprocal approximation flushes subnormals, so such pivots take an exact
    division (advisor finding: it used to give a silent NaN)."""
    n, p, t = 16, 3, 2
    rng = np.random.default_rng(5)
    xl = rng.standard_normal((n, p - 1))
    e = rng.standard_normal(n)
    e -= xl @ np.linalg.lstsq(xl, e, rcond=None)[0]  # orthogonal to X_L
    x = 1e-150 * (xl @ np.array([0.7, -1.3]) + 1e-5 * e / np.linalg.norm(e))
    y = rng.standard_normal((n, t))
    values = np.ones(n)
    with gw.Engine(n, p) as eng:
        eng.set_snp_coding("real")
        eng.set_spectrum(np.eye(n), values)
        eng.set_covariates(xl)
        eng.set_traits(y, np.zeros(t), np.ones(t), rotated=True)
        got = eng.solve_snp_slab(x.reshape(n, 1), rotated=True)
    pivot = 1e-300 * 1e-10  # |x_perp|^2: subnormal
    assert pivot < 2.2250738585072014e-308
    ref = orc.compute_grid(values, xl, x.reshape(n, 1), y, np.zeros(t), np.ones(t))
    assert np.isfinite(got).all()
    rel = np.linalg.norm(got - ref, axis=2) / np.linalg.norm(ref, axis=2)
    assert rel.max() < 1e-3, rel.max()  # the pivot itself carries ~1e-6 relative rounding
