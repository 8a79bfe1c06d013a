"""Host-side logic of the product package: argument checking and error
mapping that mirror the reference (bindings.cpp, types.cpp, grid.cpp), the
CPU eigendecomposition contract, the seeded generators, and the multi-rank
shard plan (gloo, world_size 2).  No GPU needed."""
import os

import numpy as np
import pytest

import paper_1210_7683_b200 as gw
from oracle import oracle as orc
from paper_1210_7683_b200 import datagen


def small():
    return datagen.generate(16, 3, 6, 4, seed=9)


def test_eigendecompose_contract_and_oracle_agreement():
    ds = datagen.generate(40, 3, 2, 2, seed=3)
    z, lam = gw.eigendecompose(ds["kinship"])
    assert np.all(np.diff(lam) >= 0)
    assert np.abs(z @ np.diag(lam) @ z.T - ds["kinship"]).max() < 1e-12 * np.abs(ds["kinship"]).max()
    assert np.abs(z.T @ z - np.eye(40)).max() < 1e-13
    at = np.argmax(np.abs(z), axis=0)
    assert np.all(z[at, np.arange(40)] > 0)
    zo, lo = orc.eigendecompose(ds["kinship"])
    assert np.abs(z - zo).max() < 1e-12 and np.abs(lam - lo).max() < 1e-12


def test_eigendecompose_rejects_asymmetric():
    phi = np.eye(5)
    phi[1, 3] = 0.5
    with pytest.raises(gw.NonSymmetricError):
        gw.eigendecompose(phi)
    with pytest.raises(ValueError):  # reference maps NonSymmetricError to ValueError
        gw.eigendecompose(phi)


def test_solve_grid_argument_errors():
    ds = small()
    args = (ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    with pytest.raises(ValueError, match="scheduler"):
        gw.solve_grid(*args, scheduler="bogus")
    with pytest.raises(ValueError, match="budget"):
        gw.solve_grid(*args, memory_budget=64)
    with pytest.raises(gw.InfeasibleBudgetError):
        gw.solve_grid(*args, memory_budget=64)
    with pytest.raises(gw.DimensionError, match="tile parameter nb"):
        gw.solve_grid(*args, nb=7)
    with pytest.raises(gw.DimensionError, match="tile parameter tbb"):
        gw.solve_grid(*args, tb=2, tbb=3)
    with pytest.raises(gw.DimensionError, match="one entry per trait"):
        gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"][:2], ds["sigma2"])
    with pytest.raises(gw.DimensionError, match="row counts"):
        gw.solve_grid(ds["kinship"], ds["xl"][:5], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    with pytest.raises(gw.DimensionError, match="must not exceed n"):
        gw.solve_grid(np.eye(2), np.ones((2, 2)), np.ones((2, 1)), np.ones((2, 1)), [0.5], [1.0])


def test_error_classes_mirror_reference_python_mapping():
    """bindings.cpp:232-248: NPD/Dimension/NonSymmetric/Budget -> ValueError,
    IoError -> OSError, other -> RuntimeError."""
    assert issubclass(gw.NotPositiveDefiniteError, ValueError)
    assert issubclass(gw.DimensionError, ValueError)
    assert issubclass(gw.NonSymmetricError, ValueError)
    assert issubclass(gw.InfeasibleBudgetError, ValueError)
    assert issubclass(gw.IoError, OSError)
    assert issubclass(gw.BackendError, RuntimeError)
    assert issubclass(gw.DeviceError, RuntimeError)
    e = gw.NotPositiveDefiniteError("x", 42, 6)
    assert (e.snp_index, e.trait_index) == (42, 6)


def test_status_to_exception_mapping():
    from paper_1210_7683_b200 import _native as nat
    from paper_1210_7683_b200.errors import raise_for

    st = nat.Status()
    st.code, st.snp_index, st.trait_index, st.msg = nat.GWG_NOT_POSITIVE_DEFINITE, 5, 0, b"npd"
    with pytest.raises(gw.NotPositiveDefiniteError) as e:
        raise_for(st)
    assert (e.value.snp_index, e.value.trait_index) == (5, 0)
    st.code = nat.GWG_CUDA
    with pytest.raises(gw.DeviceError):
        raise_for(st)
    st.code = nat.GWG_OK
    raise_for(st)


def test_device_working_set_is_monotone():
    a = gw.device_working_set_bytes(1000, 4, 1000, 1)
    b = gw.device_working_set_bytes(1000, 4, 1000, 100)
    assert 0 < a < b
    assert gw.device_working_set_bytes(1000, 4, 1000, 0) < a
    # the genotype path keeps W slices, S_BR and the int8 slab on top
    assert gw.device_working_set_bytes(1000, 4, 1000, 100, "genotypes") > b


def test_generator_is_deterministic_and_shaped():
    a, b = small(), small()
    for key in ("kinship", "xl", "snps", "traits", "h2", "sigma2"):
        assert np.array_equal(a[key], b[key]), key
    assert a["kinship"].shape == (16, 16) and a["xl"].shape == (16, 2)
    assert a["snps"].shape == (16, 6) and a["traits"].shape == (16, 4)
    assert not np.array_equal(a["snps"], datagen.generate(16, 3, 6, 4, seed=10)["snps"])


def test_generator_distributions_follow_baseline_json():
    ds = datagen.generate(400, 4, 300, 200, seed=5)
    assert set(np.unique(ds["snps"])) <= {0.0, 1.0, 2.0}
    assert np.all(ds["xl"][:, 0] == 1.0)  # intercept
    assert abs(ds["xl"][:, 1:].mean()) < 0.1 and abs(ds["xl"][:, 1:].std() - 1) < 0.1
    assert abs(ds["traits"].mean()) < 0.05 and abs(ds["traits"].std() - 1) < 0.05
    assert ds["h2"].min() >= 0.05 and ds["h2"].max() <= 0.95
    assert np.all(ds["sigma2"] == 1.0)
    # per-column allele frequency ~ U[0.05, 0.5]: mean genotype 2*maf in [0.1, 1.0]
    colmean = ds["snps"].mean(axis=0)
    assert colmean.min() > 0.0 and colmean.max() < 1.2
    phi = ds["kinship"]
    assert np.array_equal(phi, phi.T)
    assert np.linalg.eigvalsh(phi).min() > 1e-3 * 0.999  # + 1e-3 I
    assert abs(np.mean(np.diag(phi)) - (1.0 + 1e-3)) < 0.05  # standardized genotypes


def test_generator_columns_are_independent_of_range():
    """Counter-based: any SNP column range regenerates bit-identically (this
    is what lets each rank generate only its shard)."""
    full = datagen.genotypes(11, datagen.M_SNPS, 50, 0, 40)
    part = datagen.genotypes(11, datagen.M_SNPS, 50, 17, 9)
    assert np.array_equal(full[:, 17:26], part)
    nf = datagen.normals(11, datagen.M_TRAITS, 50, 0, 10)
    assert np.array_equal(nf[:, 3:5], datagen.normals(11, datagen.M_TRAITS, 50, 3, 2))


def _oracle_compute(shared, x, i0):
    """The per-rank solve injected into multi.solve_sharded: the oracle
    (test infrastructure) in place of the device engine."""
    from paper_1210_7683_b200.checksum import grid_checksum

    z, lam = shared["basis"].numpy(), shared["values"].numpy()
    xl, y = shared["xl"].numpy(), shared["y"].numpy()
    b = orc.compute_grid(lam, z.T @ xl, z.T @ x, z.T @ y, shared["h2"].numpy(),
                         shared["sigma2"].numpy())
    return b, grid_checksum(b, i0=i0)


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1210_7683_b200 import multi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, p, m, t = 24, 3, 21, 4

    def make_shared():  # rank 0 only: the one-off preloop
        ds = datagen.generate(n, p, 1, t, seed=4)
        z, lam = gw.eigendecompose(ds["kinship"])
        return {"basis": z, "values": lam, "xl": ds["xl"], "y": ds["traits"], "h2": ds["h2"],
                "sigma2": ds["sigma2"]}

    def load_shard(i0, i1):  # each rank generates only its own columns
        return datagen.genotypes(4, datagen.M_SNPS, n, i0, i1 - i0)

    res = multi.solve_sharded(n, p, m, t, make_shared, load_shard, _oracle_compute)
    gathered = [None] * world
    dist.all_gather_object(gathered, (res["i0"], res["i1"], res["b"]))
    if rank == 0:
        q.put((gathered, res["checksum"]))
    dist.destroy_process_group()


def test_snp_sharding_over_two_ranks_matches_single_rank():
    """The multi-GPU plan (paper_1210_7683_b200.multi, which bench.py uses):
    shard m over ranks, broadcast the shared operands once, no data-path
    collective.  Run with gloo on CPU, world size 2, through solve_sharded
    with the per-rank solve injected (the oracle here; engine_compute on the
    GPU): the shards tile [0, m) and reassemble the single-rank grid bit for
    bit, and the gathered checksum is the whole grid's."""
    import multiprocessing as mp
    import socket

    from paper_1210_7683_b200.checksum import grid_checksum

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    gathered, checksum = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert [(a, b) for a, b, _ in gathered] == [(0, 10), (10, 21)]
    sharded = np.concatenate([b for _, _, b in gathered], axis=0)
    ds = datagen.generate(24, 3, 21, 4, seed=4)
    z, lam = gw.eigendecompose(ds["kinship"])
    whole = orc.compute_grid(lam, z.T @ ds["xl"], z.T @ ds["snps"], z.T @ ds["traits"],
                             ds["h2"], np.ones(4))
    assert np.array_equal(sharded, whole)
    assert checksum == grid_checksum(whole)


def test_shard_plan_matches_device_group_formula():
    """multi.shard_bounds (torchrun ranks) and gwg_group_shards (one process,
    several GPUs) split m identically: contiguous, balanced, covering."""
    from paper_1210_7683_b200 import multi

    for m in (1, 7, 100, 100_001):
        for world in (1, 2, 3, 4, 8):
            b = multi.shard_bounds(m, world)
            assert b[0] == 0 and b[-1] == m
            sizes = np.diff(b)
            assert sizes.min() >= 0 and sizes.max() - sizes.min() <= 1
            assert multi.rank_range(m, world, world - 1) == (b[-2], b[-1])
    # weak scaling (bench.py): m per rank fixed -> rank r owns [r m, (r+1) m)
    assert multi.shard_bounds(8 * 1000, 8) == [r * 1000 for r in range(9)]


def test_empty_grids_are_dimension_errors():
    """ProblemDims::validate (types.cpp:7-17): m, t >= 1 — checked before any
    device work, like the reference."""
    ds = small()
    with pytest.raises(gw.DimensionError, match="m must be >= 1"):
        gw.solve_grid(ds["kinship"], ds["xl"], np.zeros((16, 0)), ds["traits"], ds["h2"],
                      ds["sigma2"])
    with pytest.raises(gw.DimensionError, match="t must be >= 1"):
        gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], np.zeros((16, 0)), [], [])
