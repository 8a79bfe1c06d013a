"""run_grid's streamed traversal beyond one host array: int8 genotype input
(GWG_FORMAT_I8), result sinks over rotating pinned buffers, the
order-independent device checksum, global SNP offsets (shards), the
one-process device Group, measured I/O stall, deferred trait errors, and
engine options.  Against the oracle and bit for bit against the plain
in-memory run.  References: run_grid / pipeline_run
(proj/src/grid.cpp:454-641, proj/include/gwgrid/pipeline.hpp:78-137),
write_result_cells (proj/src/stream.cpp:414-445), sampled verification
(proj/tools/gwgrid_main.cpp:336-353)."""
import os
import queue

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1210_7683_b200 as gw  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402
from tests.test_gpu_parity import assert_parity  # noqa: E402


def engine(ds, basis, values, coding="auto"):
    n, p = ds["kinship"].shape[0], ds["xl"].shape[1] + 1
    eng = gw.Engine(n, p)
    eng.set_spectrum(basis, values)
    eng.set_covariates(ds["xl"])
    eng.set_snp_coding(coding)
    eng.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
    return eng


@pytest.fixture(scope="module")
def case():
    ds = datagen.generate(300, 4, 1000, 70, seed=13)
    basis, values = gw.eigendecompose(ds["kinship"])
    with engine(ds, basis, values) as eng:
        base = eng.run_grid(ds["snps"])
    return ds, basis, values, base


@pytest.mark.parametrize("coding", ["auto", "genotypes", "real"])
def test_int8_codes_give_the_float64_bits(case, coding):
    """X_R as 1-byte codes: the same cells bit for bit as the float64 slab,
    every coding (real converts the codes to FP64 on the device)."""
    ds, basis, values, _ = case
    codes = ds["snps"].astype(np.int8)
    for mb in (0, 129):
        with engine(ds, basis, values, coding) as eng:
            want = eng.run_grid(ds["snps"], mb=mb)
            got = eng.run_grid(codes, mb=mb)
        assert np.array_equal(got, want)
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]), orc.rotate(basis, ds["snps"]),
                           orc.rotate(basis, ds["traits"]), ds["h2"], ds["sigma2"], workers=8)
    assert_parity(got, ref)


def test_int8_minus_128_is_rejected(case):
    ds, basis, values, _ = case
    codes = ds["snps"].astype(np.int8)
    codes[5, 17] = -128
    with engine(ds, basis, values) as eng:
        with pytest.raises(gw.DimensionError, match="-127, 127"):
            eng.run_grid(codes)


@pytest.mark.parametrize("layout", ["numpy", "stream"])
@pytest.mark.parametrize("ring", [2, 3])
def test_sink_receives_every_cell_once(case, layout, ring):
    """Results through a sink over rotating pinned buffers: every slab once,
    in order, global i0, slab-local layout; together bitwise the in-memory
    grid."""
    ds, basis, values, base = case
    m = base.shape[0]
    got = np.full_like(base, np.nan)
    seen = []

    def sink(i0, cells):
        seen.append((i0, cells.shape))
        rows = cells.shape[0] if layout == "numpy" else cells.shape[1]
        got[i0:i0 + rows] = cells if layout == "numpy" else cells.transpose(1, 0, 2)

    with engine(ds, basis, values) as eng:
        assert eng.run_grid(ds["snps"], mb=130, layout=layout, sink=sink, ring=ring) is None
    assert [s[0] for s in seen] == list(range(0, m, 130))
    assert np.array_equal(got, base)


def test_sink_error_aborts_the_run(case):
    ds, basis, values, _ = case

    class Boom(Exception):
        pass

    def sink(i0, cells):
        if i0 >= 200:
            raise Boom()

    with engine(ds, basis, values) as eng:
        with pytest.raises(Boom):
            eng.run_grid(ds["snps"], mb=100, sink=sink)
        # the engine stays usable
        assert np.array_equal(eng.run_grid(ds["snps"]), case[3])


def test_checksum_is_order_independent_and_tied_to_bits(case):
    """Device checksum == host recomputation from the downloaded bits; equal
    across slab widths, layouts, input formats, buffering and shard splits
    (i0 offsets); sensitive to the inputs."""
    ds, basis, values, base = case
    want = gw.grid_checksum(base)
    runs = [dict(mb=0), dict(mb=1), dict(mb=77), dict(mb=333, layout="stream"),
            dict(mb=128, double_buffer=False)]
    with engine(ds, basis, values) as eng:
        for kw in runs:
            eng.reset_counters()
            eng.run_grid(ds["snps"], checksum=True, **kw)
            c = eng.counters()
            assert c["checksum"] == want, kw
            assert c["checksum_cells"] == base.shape[0] * base.shape[1]
        eng.reset_counters()
        eng.run_grid(ds["snps"].astype(np.int8), checksum=True)
        assert eng.counters()["checksum"] == want
        # shards with global offsets sum to the whole grid's checksum
        eng.reset_counters()
        for a, b in ((0, 1), (1, 400), (400, 1000)):
            part = eng.run_grid(np.asfortranarray(ds["snps"][:, a:b]), checksum=True, i0=a)
            assert np.array_equal(part, base[a:b])
        assert eng.counters()["checksum"] == want
        # another trait set changes it
        eng.set_traits(ds["traits"][:, ::-1].copy(), ds["h2"][::-1].copy(), ds["sigma2"])
        eng.reset_counters()
        eng.run_grid(ds["snps"], checksum=True)
        assert eng.counters()["checksum"] != want


def test_shard_error_coordinates_are_global(case):
    ds, basis, values, _ = case
    snps = ds["snps"].copy()
    snps[:, 612] = 0.0
    with engine(ds, basis, values) as eng:
        with pytest.raises(gw.NotPositiveDefiniteError) as e:
            eng.run_grid(np.asfortranarray(snps[:, 600:700]), i0=600)
    assert (e.value.snp_index, e.value.trait_index) == (612, 0)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
def test_device_group_matches_one_engine(case, devices):
    """The one-process multi-GPU driver (gwg_group_*): shared operands
    broadcast device-to-device, m sharded into contiguous ranges, one host
    thread per device.  Bitwise the single engine's grid for 2 and 4 shards
    (here all on GPU 0: the shards do not wait on each other), any layout,
    int8 input, with the single engine's checksum and global error
    coordinates."""
    ds, basis, values, base = case
    n, p = 300, 4
    with gw.Group(n, p, devices) as g:
        bounds = g.shards(1000)
        assert bounds[0] == 0 and bounds[-1] == 1000 and len(bounds) == len(devices) + 1
        g.set_spectrum(basis, values)
        g.set_covariates(ds["xl"])
        g.set_traits(ds["traits"], ds["h2"], ds["sigma2"])
        b = g.run_grid(ds["snps"], checksum=True, mb=97)
        assert np.array_equal(b, base)
        assert g.counters()["checksum"] == gw.grid_checksum(base)
        s = g.run_grid(ds["snps"].astype(np.int8), layout="stream")
        assert np.array_equal(s.transpose(1, 0, 2), base)
        got = np.empty_like(base)

        def sink(i0, cells):  # called from one thread per device
            got[i0:i0 + cells.shape[0]] = cells

        g.run_grid(ds["snps"], sink=sink, mb=64)
        assert np.array_equal(got, base)
        snps = ds["snps"].copy()
        snps[:, [900, 620]] = 0.0
        with pytest.raises(gw.NotPositiveDefiniteError) as e:
            g.run_grid(snps)
        assert (e.value.snp_index, e.value.trait_index) == (620, 0)
    res = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                        ds["sigma2"], devices=devices)
    ref = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                        ds["sigma2"])
    assert np.array_equal(res["b"], ref["b"])


def test_pipeline_stall_is_measured(case):
    """io_stall_seconds / stall_fraction are measured (compute-stream gaps +
    tail), not constants: positive with a serialised pipeline, and no larger
    than the wall time."""
    ds = case[0]
    args = (ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"])
    serial = gw.solve_grid(*args, mb=100, double_buffer=False)["counters"]
    assert 0.0 < serial["io_stall_seconds"] <= serial["loops_wall_seconds"]
    assert 0.0 < serial["stall_fraction"] <= 1.0
    assert serial["preloop_wall_seconds"] > 0.0


def test_trait_failure_is_reported_by_the_next_sync():
    """gwg_set_traits queues its work without a host round trip: a weight
    floor failure (-1, j) surfaces at the next synchronising call, ahead of
    any cell error, from host and device operands alike."""
    n = 8
    phi = np.diag(np.arange(n) - 0.5)
    basis, values = gw.eigendecompose(phi)
    rng = np.random.default_rng(3)
    h2 = np.zeros(5)
    h2[3] = 0.9
    y = rng.standard_normal((n, 5))
    x = rng.integers(0, 3, (n, 4)).astype(float)
    for dev in (False, True):
        with gw.Engine(n, 2) as eng:
            eng.set_spectrum(basis, values)
            eng.set_covariates(np.ones((n, 1)))
            args = (y, h2, np.ones(5))
            if dev:
                args = tuple(torch.from_numpy(np.asarray(a)).cuda() for a in args)
            eng.set_traits(*args)
            with pytest.raises(gw.NotPositiveDefiniteError) as e:
                eng.synchronize()
            assert (e.value.snp_index, e.value.trait_index) == (-1, 3)
            with pytest.raises(gw.NotPositiveDefiniteError) as e:
                eng.solve_snp_slab(x)
            assert (e.value.snp_index, e.value.trait_index) == (-1, 3)


def test_device_out_must_match_dtype_and_device(case):
    ds, basis, values, _ = case
    x = torch.from_numpy(np.asarray(ds["snps"][:, :10])).cuda()
    with engine(ds, basis, values) as eng:
        with pytest.raises(gw.DimensionError, match="float64"):
            eng.solve_snp_slab(x, out=torch.empty((10, 70, 4), device="cuda"))
        with pytest.raises(gw.DimensionError, match="float64"):
            eng.solve_snp_slab(x.float())
        out = torch.empty((10, 70, 4), dtype=torch.float64, device="cuda")
        eng.solve_snp_slab(x, out=out)
        assert np.array_equal(out.cpu().numpy(), case[3][:10])


def test_options_replace_environment_switches(case, monkeypatch):
    """Numerics depend on explicit options only: the round-1 environment
    switches are ignored; every option value round-trips and is validated."""
    ds, basis, values, base = case
    for var in ("GWG_SBR_DIRECT", "GWG_REAL_SPLIT", "GWG_SPLIT", "GWG_I8_CLUSTER", "GWG_SBR_CFG"):
        monkeypatch.setenv(var, "1")
    with engine(ds, basis, values) as eng:
        assert np.array_equal(eng.run_grid(ds["snps"]), base)
        for name, value in (("split", 0), ("sbr_direct", 1), ("real_split", 0),
                            ("i8_cluster", 3), ("sbr_cfg", 2)):
            eng.set_option(name, value)
            assert eng.get_option(name) == value
        b = eng.run_grid(ds["snps"])
        rel = np.linalg.norm(b - base, axis=2) / np.linalg.norm(base, axis=2)
        assert rel.max() < 1e-11
        with pytest.raises(gw.DimensionError):
            eng.set_option("i8_cluster", 7)
        with pytest.raises(gw.DimensionError):
            eng.set_option("nope", 1)


def test_config3_shape_reduced_m_checksum_and_spot_checks():
    """BASELINE configs[3] (n=1000, p=4, t=100,000) at full t with m reduced to
    640 SNPs (6.4e7 cells): results stream through a sink over rotating pinned
    buffers and are never held whole; the device checksum agrees across two
    slab widths and with a sink-side host recomputation, and seeded random
    cells match the oracle and the independent Cholesky route."""
    n, p, m, t = 1000, 4, 640, 100_000
    ds = datagen.generate(n, p, m, t, seed=33)
    basis, values = gw.eigendecompose(ds["kinship"])
    rng = np.random.default_rng(7)
    ii, jj = rng.integers(0, m, 24), rng.integers(0, t, 24)
    sums = []
    picked = {}
    host_sum = [0]

    def sink(i0, cells):
        host_sum[0] = (host_sum[0] + gw.grid_checksum(cells, i0=i0)) & (2**64 - 1)
        for k, (i, j) in enumerate(zip(ii, jj)):
            if i0 <= i < i0 + cells.shape[0]:
                picked[k] = cells[i - i0, j].copy()

    with engine(ds, basis, values) as eng:
        for mb in (128, 256):
            eng.reset_counters()
            host_sum[0] = 0
            eng.run_grid(ds["snps"].astype(np.int8), sink=sink, checksum=True, mb=mb, ring=3)
            c = eng.counters()
            assert c["checksum_cells"] == m * t
            assert c["checksum"] == host_sum[0]
            sums.append(c["checksum"])
    assert sums[0] == sums[1]
    got = np.stack([picked[k] for k in range(len(ii))])
    cols = np.unique(ii)
    pos = {c: k for k, c in enumerate(cols)}
    tcols = np.unique(jj)
    tpos = {c: k for k, c in enumerate(tcols)}
    ref = orc.compute_grid(values, orc.rotate(basis, ds["xl"]),
                           orc.rotate(basis, ds["snps"][:, cols]),
                           orc.rotate(basis, ds["traits"][:, tcols]), ds["h2"][tcols],
                           ds["sigma2"][tcols], workers=8)
    want = np.stack([ref[pos[i], tpos[j]] for i, j in zip(ii, jj)])
    assert_parity(got, want)
    chol = orc.cholesky_cells(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"],
                              ds["sigma2"], ii[:6], jj[:6])
    assert (np.linalg.norm(got[:6] - chol, axis=1) / np.linalg.norm(chol, axis=1)).max() < 1e-10


def test_device_output_solves_are_asynchronous_with_deferred_errors(case):
    """A device-output solve_snp_slab queues its work and returns; errors of
    every slab since the last synchronising call surface there, the first
    failing cell in trait-major order over all of them, with global
    coordinates; torch work after the call is ordered after it."""
    ds, basis, values, base = case
    snps = ds["snps"].copy()
    snps[:, 733] = 0.0
    snps[:, 120] = 0.0
    x = torch.from_numpy(snps).cuda()
    out = torch.empty((1000, 70, 4), dtype=torch.float64, device="cuda")
    with engine(ds, basis, values) as eng:
        eng.solve_snp_slab(x[:, 500:].contiguous(), out=out[500:], i0=500)  # no raise yet
        eng.solve_snp_slab(x[:, :500].contiguous(), out=out[:500], i0=0)
        with pytest.raises(gw.NotPositiveDefiniteError) as e:
            eng.synchronize()
        assert (e.value.snp_index, e.value.trait_index) == (120, 0)
        eng.synchronize()  # the epoch closed: nothing left to report
        good = torch.from_numpy(ds["snps"]).cuda()
        eng.solve_snp_slab(good, out=out)
        got = out.cpu().numpy()  # torch's stream waits for the engine
        eng.synchronize()
    assert np.array_equal(got, base)


def test_trait_side_stream_interleavings(case):
    """On the split path gwg_set_traits queues its work on the engine's side
    stream and the SNP rotation joins it (set_traits_impl, split_build_ahead):
    whatever runs in between — a second set_traits, new covariates, an option
    change, a host run_grid, an error read — sees the traits of the last
    set_traits, bit for bit what a fresh engine computes."""
    ds, basis, values, base = case
    rng = np.random.default_rng(5)
    y2 = rng.standard_normal(ds["traits"].shape)
    h2b = rng.uniform(0.1, 0.9, ds["h2"].shape)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    x = dev(ds["snps"])
    with gw.Engine(ds["kinship"].shape[0], 4) as fresh:
        fresh.set_spectrum(basis, values)
        fresh.set_covariates(ds["xl"])
        fresh.set_snp_coding("genotypes")
        fresh.set_traits(y2, h2b, ds["sigma2"])
        ref2 = fresh.run_grid(ds["snps"])
    with engine(ds, basis, values, coding="genotypes") as eng:
        first = eng.run_grid(ds["snps"])
        assert np.array_equal(first, base)
        # two trait sets back to back on the device: the second wins
        eng.set_traits(dev(ds["traits"]), dev(ds["h2"]), dev(ds["sigma2"]))
        eng.set_traits(dev(y2), dev(h2b), dev(ds["sigma2"]))
        out = torch.empty((ds["snps"].shape[1], 70, 4), dtype=torch.float64, device="cuda")
        eng.solve_snp_slab(x, out=out)
        eng.synchronize()
        assert np.array_equal(out.cpu().numpy(), ref2)
        # device traits, then a host run_grid straight away
        eng.set_traits(dev(ds["traits"]), dev(ds["h2"]), dev(ds["sigma2"]))
        assert np.array_equal(eng.run_grid(ds["snps"]), base)
        # device traits, an option round trip and new (equal) covariates in between
        eng.set_traits(dev(y2), dev(h2b), dev(ds["sigma2"]))
        eng.set_option("i8_cluster", 1)
        eng.set_covariates(ds["xl"])
        eng.set_traits(dev(y2), dev(h2b), dev(ds["sigma2"]))
        eng.set_option("i8_cluster", 0)
        out2 = torch.empty_like(out)
        eng.solve_snp_slab(x, out=out2)
        got = out2.cpu().numpy()  # torch's stream is ordered after the engine
        assert np.array_equal(got, ref2)


def _nccl_rank_worker(port, q):
    """One torch.distributed rank on cuda:0 with the NCCL backend (a one-GPU
    box can host a world of one): multi.solve_sharded with the device engine
    as the per-rank solve — the code path of every rank of bench.py --gpus N."""
    import torch
    import torch.distributed as dist

    from paper_1210_7683_b200 import multi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1",
                      LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    n, p, m, t = 200, 4, 700, 40

    def make_shared():
        ds = datagen.generate(n, p, 1, t, seed=12)
        z, lam = gw.eigendecompose(ds["kinship"])
        return {"basis": z, "values": lam, "xl": ds["xl"], "y": ds["traits"], "h2": ds["h2"],
                "sigma2": ds["sigma2"]}

    def load_shard(i0, i1):
        return datagen.genotypes(12, datagen.M_SNPS, n, i0, i1 - i0)

    res = multi.solve_sharded(n, p, m, t, make_shared, load_shard, multi.engine_compute(0),
                              device=torch.device("cuda", 0))
    q.put((res["i0"], res["i1"], np.asarray(res["b"]), res["checksum"]))
    dist.destroy_process_group()


def test_solve_sharded_with_the_engine_under_nccl():
    """multi.solve_sharded + multi.engine_compute under an NCCL process group
    on the GPU (world size 1): NCCL broadcasts of the shared operands into
    HBM, the engine fed from those device tensors, the checksum all-gather —
    equal, bit for bit, to the single-engine grid and its checksum."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_rank_worker, args=(port, q))
    pr.start()
    got = None
    for _ in range(300):  # a crashed worker fails the test at once, not after the timeout
        try:
            got = q.get(timeout=1)
            break
        except queue.Empty:
            if not pr.is_alive():
                break
    pr.join(timeout=120)
    assert got is not None and pr.exitcode == 0, f"worker exit code {pr.exitcode}"
    i0, i1, b, checksum = got
    assert (i0, i1) == (0, 700)
    ds = datagen.generate(200, 4, 700, 40, seed=12)
    whole = gw.solve_grid(ds["kinship"], ds["xl"], ds["snps"], ds["traits"], ds["h2"], ds["sigma2"],
                          checksum=True)
    assert np.array_equal(b, whole["b"])
    assert checksum == whole["counters"]["checksum"] == gw.grid_checksum(whole["b"])
