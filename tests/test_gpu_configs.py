"""BASELINE.json configs 2-4 at full n, p, t on the device, against the oracle
on seeded SNP x trait samples (the full m would take hours on the CPU; cells
are independent, so a sub-grid is exactly the corresponding part of the full
grid — the device results are bitwise independent of slab geometry).

config 2: n=10,000, p=4, t=1,000, kinship from s=20,000 (eigendecomposition on
          the device, shared with the oracle like BASELINE.md prescribes)
config 3: n=1,000, p=4, t=100,000 (the paper's largest shape)
config 4: n=2,000, p=20, t=2,000 (20x20 systems)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1210_7683_b200 as gw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402
from tests.test_gpu_parity import assert_parity, metrics  # noqa: E402


def run_config(n, p, t, s, m_dev, m_orc, t_orc, seed, device_eig, coding="real"):
    phi = datagen.kinship(seed, n, s)
    if device_eig:
        basis, values = gw.eigendecompose(phi, device=0)
    else:
        basis, values = gw.eigendecompose(phi)
    xl = datagen.covariates(seed, n, p)
    traits = datagen.normals(seed, datagen.M_TRAITS, n, 0, t)
    h2 = datagen.uniform(seed, datagen.M_H2, t, 0.05, 0.95)
    s2 = np.ones(t)
    col0 = 123_456  # a slab from the middle of the SNP axis
    snps = datagen.genotypes(seed, datagen.M_SNPS, n, col0, m_dev)
    with gw.Engine(n, p) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(xl)
        eng.set_snp_coding(coding)
        eng.set_traits(traits, h2, s2)
        b = eng.run_grid(snps)
        b2 = eng.run_grid(snps, mb=37)
    assert not np.isnan(b).any()
    # checksum of checksums: two slab widths agree bit for bit
    assert np.array_equal(b.view(np.uint64).sum(axis=(1, 2)), b2.view(np.uint64).sum(axis=(1, 2)))
    rng = np.random.default_rng(seed)
    ii = np.sort(rng.choice(m_dev, m_orc, replace=False))
    jj = np.sort(rng.choice(t, t_orc, replace=False))
    ref = orc.compute_grid(values, orc.rotate(basis, xl), orc.rotate(basis, snps[:, ii]),
                           orc.rotate(basis, traits[:, jj]), h2[jj], s2[jj], workers=16)
    got = b[np.ix_(ii, jj)]
    assert_parity(got, ref)
    return metrics(got, ref)


@pytest.mark.parametrize("coding", ["real", "genotypes"])
def test_config2_large_n(coding):
    print(run_config(10_000, 4, 1000, 20_000, 600, 150, 100, 2, device_eig=True, coding=coding))


@pytest.mark.parametrize("coding", ["real", "genotypes"])
def test_config3_many_traits(coding):
    print(run_config(1000, 4, 100_000, 2000, 300, 100, 1500, 3, device_eig=False, coding=coding))


@pytest.mark.parametrize("coding", ["real", "genotypes"])
def test_config4_many_covariates(coding):
    print(run_config(2000, 20, 2000, 2000, 700, 200, 200, 4, device_eig=False, coding=coding))


def test_split_k_g_gemm_is_slab_invariant_and_matches_oracle():
    """From K >= 2048 the S_BR stage's G = (X'.X')^T E GEMM splits K by n alone
    (launch_sbr_stage); n = 2080 gives 65 K-chunks -> two parts of 33 with one
    zero-padded chunk.  Results: bitwise independent of the slab width (the
    split never depends on the slab) and equal to the oracle to rounding, on
    both codings (the FP64 path factorises S_BR too for t >= 256)."""
    from oracle import oracle as orc
    from tests.test_gpu_parity import assert_parity

    n, p, m, t = 2080, 3, 700, 260
    ds = datagen.generate(n, p, m, t, seed=41)
    basis, values = gw.eigendecompose(ds["kinship"])
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                           orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)
    for coding in ("genotypes", "real"):
        with gw.Engine(n, p) as eng:
            eng.set_spectrum(basis, values)
            eng.set_covariates(ds["xl"])
            eng.set_snp_coding(coding)
            eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
            whole = eng.run_grid(ds["snps"], mb=700)
            for mb in (100, 333):
                assert np.array_equal(eng.run_grid(ds["snps"], mb=mb), whole), (coding, mb)
        assert_parity(whole, ref)
