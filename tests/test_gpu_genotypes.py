"""Genotype coding: the exact int8 tcgen05 rotation and the split grid (S_BR on
DMMA, linear terms exactly on int8 tcgen05 + the solve) against the all-FP64
path and the oracle, for every p and both layouts; the device-side input
check; failure semantics; slab invariance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1210_7683_b200 as gw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402
from tests.test_gpu_parity import assert_parity  # noqa: E402


def run(ds, basis, values, coding, options=None, **kw):
    n, p = ds["kinship"].shape[0], ds["xl"].shape[1] + 1
    with gw.Engine(n, p) as eng:
        for name, value in (options or {}).items():
            eng.set_option(name, value)
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        return eng.run_grid(ds["snps"], **kw)


@pytest.mark.parametrize("n,p,m,t", [(1000, 4, 3000, 64), (257, 4, 333, 37), (130, 1, 70, 9),
                                     (300, 12, 129, 17), (64, 3, 5, 3), (2000, 20, 300, 20)])
def test_genotype_path_matches_real_path_and_oracle(n, p, m, t):
    ds = datagen.generate(n, p, m, t, seed=n + 3 * p)
    basis, values = gw.eigendecompose(ds["kinship"])
    bg = run(ds, basis, values, "genotypes")
    br = run(ds, basis, values, "real")
    assert not np.isnan(bg).any()
    rel = np.linalg.norm(bg - br, axis=2) / np.linalg.norm(br, axis=2)
    assert rel.max() < 1e-11, rel.max()
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                           orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)
    assert_parity(bg, ref)


@pytest.mark.parametrize("p", list(range(1, 33)))
def test_split_grid_every_p_and_layout(p):
    """The split grid (S_BR on DMMA, exact int8 linear terms + solve) for every
    compiled p, both result layouts, against the all-FP64 path."""
    n, m, t = 96 + p, 150, 11
    ds = datagen.generate(n, p, m, t, seed=100 + p)
    basis, values = gw.eigendecompose(ds["kinship"])
    bg = run(ds, basis, values, "genotypes")
    br = run(ds, basis, values, "real")
    assert not np.isnan(bg).any()
    rel = np.linalg.norm(bg - br, axis=2) / np.linalg.norm(br, axis=2)
    assert rel.max() < 1e-10, rel.max()
    bs = run(ds, basis, values, "genotypes", layout="stream", mb=64)
    assert np.array_equal(bs.transpose(1, 0, 2), bg)


def test_split_grid_failure_semantics_match_fp64_path():
    """A zero SNP column makes every cell of that SNP singular: NaN results and
    NotPositiveDefiniteError at the smallest (trait, SNP) key, as in the
    all-FP64 kernel."""
    ds = datagen.generate(120, 4, 40, 5, seed=3)
    snps = ds["snps"].copy()
    snps[:, 17] = 0.0
    ds2 = dict(ds, snps=snps)
    basis, values = gw.eigendecompose(ds["kinship"])
    errs = []
    for coding in ("genotypes", "real"):
        with pytest.raises(gw.NotPositiveDefiniteError) as e:
            run(ds2, basis, values, coding)
        errs.append((e.value.snp_index, e.value.trait_index))
    assert errs[0] == errs[1] == (17, 0)


def test_genotype_path_bitwise_invariant_to_slabs():
    ds = datagen.generate(300, 4, 777, 30, seed=9)
    basis, values = gw.eigendecompose(ds["kinship"])
    base = run(ds, basis, values, "genotypes")
    for mb in (1, 64, 300, 777):
        assert np.array_equal(base, run(ds, basis, values, "genotypes", mb=mb))


def test_genotype_check_rejects_non_integer_codes():
    ds = datagen.generate(64, 3, 10, 3, seed=2)
    snps = ds["snps"].copy()
    snps[5, 4] = 0.5
    ds2 = dict(ds, snps=snps)
    basis, values = gw.eigendecompose(ds["kinship"])
    with pytest.raises(gw.DimensionError, match="genotype"):
        run(ds2, basis, values, "genotypes")
    snps[5, 4] = 300.0
    with pytest.raises(gw.DimensionError, match="genotype"):
        run(dict(ds, snps=snps), basis, values, "genotypes")
    # the real-valued path accepts them
    assert np.isfinite(run(ds2, basis, values, "real")).all()


@pytest.mark.parametrize("coding", ["genotypes", "real"])
@pytest.mark.parametrize("layout", ["numpy", "stream"])
@pytest.mark.parametrize("offset", [0, 1, 2])  # doubles: 1 = 8-byte aligned only (no TMA stores)
def test_device_output_stays_inside_its_buffer(coding, layout, offset):
    """Results written straight into a device tensor that is a window of a larger
    sentinel-filled buffer: every cell written, nothing outside the window
    touched (TMA stores clip at the tensor edges; misaligned windows take the
    direct-store path)."""
    n, p, m, t = 150, 4, 203, 27
    ds = datagen.generate(n, p, m, t, seed=77)
    basis, values = gw.eigendecompose(ds["kinship"])
    ref = run(ds, basis, values, coding)
    size = m * t * p
    guard = 4096
    buf = torch.full((size + 2 * guard,), -7.25, dtype=torch.float64, device="cuda")
    shape = (m, t, p) if layout == "numpy" else (t, m, p)
    out = buf[guard + offset: guard + offset + size].view(shape)
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding(coding)
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        x = torch.from_numpy(np.ascontiguousarray(ds["snps"].T)).cuda().t()
        eng.solve_snp_slab(x, out=out, layout=layout)
        torch.cuda.synchronize()
    host = buf.cpu().numpy()
    assert np.all(host[:guard + offset] == -7.25)
    assert np.all(host[guard + offset + size:] == -7.25)
    got = out.cpu().numpy()
    if layout == "stream":
        got = got.transpose(1, 0, 2)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n", [151, 152])  # odd n: padded leading dimension on the device
@pytest.mark.parametrize("offset", [0, 1])  # 1: an 8-byte-aligned device operand
def test_device_snp_operand_alignment_and_odd_n(n, offset):
    p, m, t = 3, 77, 13
    ds = datagen.generate(n, p, m, t, seed=n + offset)
    basis, values = gw.eigendecompose(ds["kinship"])
    ref = run(ds, basis, values, "genotypes")
    flat = torch.zeros(n * m + 8, dtype=torch.float64, device="cuda")
    x = flat[offset: offset + n * m].view(m, n)
    x.copy_(torch.from_numpy(np.ascontiguousarray(ds["snps"].T)))
    out = torch.empty((m, t, p), dtype=torch.float64, device="cuda")
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding("genotypes")
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        eng.solve_snp_slab(x.t(), out=out)
        torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("case", ["config", "edge_h", "wide_spectrum"])
def test_low_rank_sbr_matches_direct_contraction(case):
    """S_BR = ((X'.X')^T E) F (positive exponential sum, csrc/expsum.cpp)
    against the direct DMMA contraction (X'.X')^T D (GWG_OPT_SBR_DIRECT) and
    the oracle, including h2 = 0 (D constant), h2 = 1 and a spectrum spanning
    nine decades."""
    n, p, m, t = 400, 4, 500, 40
    ds = datagen.generate(n, p, m, t, seed=41)
    basis, values = gw.eigendecompose(ds["kinship"])
    h2 = ds["h2"].copy()
    if case == "edge_h":
        h2[:6] = [0.0, 1.0, 1e-9, 1 - 1e-9, 0.5, 0.0]
    if case == "wide_spectrum":
        values = np.geomspace(1e-7, 1e2, n)
    ds = dict(ds, h2=h2)
    b_low = run(ds, basis, values, "genotypes")
    b_dir = run(ds, basis, values, "genotypes", options={"sbr_direct": 1})
    assert not np.isnan(b_low).any()
    rel = np.linalg.norm(b_low - b_dir, axis=2) / np.linalg.norm(b_dir, axis=2)
    assert rel.max() < 1e-11, rel.max()
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                           orc.rotate(basis, ds["traits"]), h2, ds["sigma2"], workers=8)
    assert_parity(b_low, ref)


def test_low_rank_sbr_is_used_and_falls_back():
    """The engine takes the factorised S_BR on BASELINE-like inputs (two
    gls_sbr launches per slab instead of one) and the direct contraction
    when D is outside the factorisation's range: h2 = 3, sigma2 = -1 and a
    spectrum in [0.1, 0.6] give weights sigma2 (h2 lambda + 1 - h2) > 0 that
    the reference accepts, but h2 lambda + 1 - h2 < 0 everywhere."""
    ds = datagen.generate(200, 3, 100, 8, seed=5)
    basis, values = gw.eigendecompose(ds["kinship"])
    n, p, t = 200, 3, 8

    def launches(values, h2, sigma2, direct=0):
        with gw.Engine(n, p) as eng:
            eng.set_option("sbr_direct", direct)
            eng.set_spectrum(basis, values)
            eng.set_covariates(ds["xl"])
            eng.set_snp_coding("genotypes")
            eng.set_traits(ds["traits"], h2, sigma2)
            eng.run_grid(ds["snps"])  # builds the trait operands
            eng.reset_counters()
            b = eng.run_grid(ds["snps"])
            return eng.counters()["kernel_launches"], b

    odd = (np.linspace(0.1, 0.6, n), np.full(t, 3.0), np.full(t, -1.0))
    k_low, b_low = launches(values, ds["h2"], ds["sigma2"])
    k_odd, b_odd = launches(*odd)
    k_dir, b_dir = launches(values, ds["h2"], ds["sigma2"], direct=1)
    k_odd_dir, b_odd_dir = launches(*odd, direct=1)
    assert k_low == k_dir + 1 and k_odd == k_odd_dir == k_dir
    rel = np.linalg.norm(b_low - b_dir, axis=2) / np.linalg.norm(b_dir, axis=2)
    assert rel.max() < 1e-11, rel.max()
    assert np.array_equal(b_odd, b_odd_dir)
    ref = orc.compute_grid(odd[0], orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                           orc.rotate(basis, ds["traits"]), odd[1], odd[2], workers=8)
    assert_parity(b_odd, ref)


@pytest.mark.parametrize("n,p,m,t", [(200, 4, 300, 20), (1000, 4, 1000, 64), (300, 12, 129, 17),
                                     (257, 20, 333, 7), (300, 13, 200, 20)])
def test_int8_kernel_variants_bitwise_identical(n, p, m, t):
    """Every int8 launch geometry (GWG_OPT_I8_CLUSTER: 1 single CTAs, 2 CTA pairs
    on two SNP tiles multicasting B, 3 CTA pairs on two W tiles multicasting
    the SNP tile, 4 CTA pairs running one cta_group::2 MMA with half of the
    slice tile each, 5 2 x 2 clusters multicasting halves of both operands,
    odd tile counts on both axes included) gives the same bits: the int32
    slice products are exact and the recombination order fixed."""
    ds = datagen.generate(n, p, m, t, seed=n + p)
    basis, values = gw.eigendecompose(ds["kinship"])
    out = {}
    for cl in ("1", "2", "3", "4", "5"):
        out[cl] = run(ds, basis, values, "genotypes", options={"i8_cluster": int(cl)})
    assert not np.isnan(out["2"]).any()
    for cl in ("2", "3", "4", "5"):
        assert np.array_equal(out["1"], out[cl]), cl


def test_auto_coding_picks_the_path_per_slab():
    """GWG_SNP_AUTO (the engine default): a slab of integer codes takes the
    genotype path, a slab with any other value the FP64 path — both queued,
    gated on the device check, no error.  Slab by slab the results are those
    of the explicit coding, bit for bit."""
    n, p, m, t = 300, 4, 400, 23
    ds = datagen.generate(n, p, m, t, seed=77)
    basis, values = gw.eigendecompose(ds["kinship"])
    snps = ds["snps"].copy()
    snps[7, 250] += 0.25  # SNP 250 lies in the third 100-column slab
    ds2 = dict(ds, snps=snps)
    auto = run(ds2, basis, values, "auto", mb=100)
    geno = run(ds, basis, values, "genotypes", mb=100)
    real = run(ds2, basis, values, "real", mb=100)
    assert not np.isnan(auto).any()
    assert np.array_equal(auto[:200], geno[:200])
    assert np.array_equal(auto[300:], geno[300:])
    assert np.array_equal(auto[200:300], real[200:300])
    # the default engine coding is auto
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        assert np.array_equal(eng.run_grid(ds["snps"], mb=100), geno)


@pytest.mark.parametrize("t", [23, 300])
def test_auto_coding_first_slab_non_code(t):
    """GWG_SNP_AUTO when the FIRST slab after set_traits holds a non-code
    value and every later slab codes: the trait operands of the genotype path
    (W, its slices, E/F) are built ungated on the first slab, so the later
    slabs get the explicit genotype coding's bits (advisor finding: they used
    to be built under the first slab's FP64 verdict and left stale)."""
    n, p, m = 300, 4, 400
    ds = datagen.generate(n, p, m, t, seed=78)
    basis, values = gw.eigendecompose(ds["kinship"])
    snps = ds["snps"].copy()
    snps[3, 10] += 0.5  # first 100-column slab is real-valued
    ds2 = dict(ds, snps=snps)
    auto = run(ds2, basis, values, "auto", mb=100)
    geno = run(ds, basis, values, "genotypes", mb=100)
    real = run(ds2, basis, values, "real", mb=100)
    assert not np.isnan(auto).any()
    assert np.array_equal(auto[:100], real[:100])
    assert np.array_equal(auto[100:], geno[100:])
    # the same through solve_snp_slab, slab by slab (the verdict word is reset
    # before each slab's rotation)
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        parts = [eng.solve_snp_slab(np.asfortranarray(snps[:, a:a + 100]), i0=a)
                 for a in range(0, m, 100)]
    assert np.array_equal(np.concatenate(parts), auto)


@pytest.mark.parametrize("p", [1, 4, 12, 20])
def test_fp64_path_factorised_sbr_matches_fused(p):
    """The all-FP64 path with t >= 256 takes S_BR from the factorised GEMMs and
    runs the grid kernel without the D column (GridCfg::EXT); GWG_OPT_REAL_SPLIT = 0
    keeps the single fused kernel.  Same cells to rounding, both against the
    oracle, and bitwise independent of the slab width."""
    n, m, t = 200, 150, 300
    ds = datagen.generate(n, p, m, t, seed=200 + p)
    basis, values = gw.eigendecompose(ds["kinship"])
    split = run(ds, basis, values, "real")
    assert np.array_equal(split, run(ds, basis, values, "real", mb=37))
    fused = run(ds, basis, values, "real", options={"real_split": 0})
    rel = np.linalg.norm(split - fused, axis=2) / np.linalg.norm(fused, axis=2)
    assert rel.max() < 1e-11, rel.max()
    ii = np.arange(0, m, 7)
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"][:, ii]),
                           orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)
    assert_parity(split[ii], ref)


@pytest.mark.parametrize("p", [3, 9, 12, 13, 21])
def test_split_grid_tma_row_stores(p):
    """Result rows that are not whole 128-byte chunks leave through one
    unswizzled TMA box per warp tile (odd rows keep their first or last
    double out of the box, whichever keeps the box start 16-byte aligned);
    t even makes the numpy layout TMA-storable.  Against the FP64 path and
    the stream layout's direct stores."""
    n, m, t = 150, 300, 20
    ds = datagen.generate(n, p, m, t, seed=300 + p)
    basis, values = gw.eigendecompose(ds["kinship"])
    bg = run(ds, basis, values, "genotypes")
    br = run(ds, basis, values, "real")
    rel = np.linalg.norm(bg - br, axis=2) / np.linalg.norm(br, axis=2)
    assert not np.isnan(bg).any() and rel.max() < 1e-10, rel.max()
    bs = run(ds, basis, values, "genotypes", layout="stream", mb=64)
    assert np.array_equal(bs.transpose(1, 0, 2), bg)


def test_genotype_coding_prerotated_slab_builds_panels_on_demand():
    """Explicit genotype coding skips the FP64 grid's operand panels at
    gwg_set_traits; a pre-rotated slab (always the FP64 path) builds them on
    demand and gets the FP64 path's result."""
    n, p, m, t = 160, 4, 90, 12
    ds = datagen.generate(n, p, m, t, seed=91)
    basis, values = gw.eigendecompose(ds["kinship"])
    xr = np.asfortranarray(basis.T @ ds["snps"])
    out = {}
    for coding in ("genotypes", "real"):
        with gw.Engine(n, p) as eng:
            eng.set_spectrum(basis, values)
            eng.set_covariates(ds["xl"])
            eng.set_snp_coding(coding)
            eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
            out[coding] = eng.solve_snp_slab(xr, rotated=True)
    assert not np.isnan(out["genotypes"]).any()
    assert np.array_equal(out["genotypes"], out["real"])
