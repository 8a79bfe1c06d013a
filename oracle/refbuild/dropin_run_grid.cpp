// dropin_run_grid.cpp — TEST INFRASTRUCTURE ONLY: the drop-in, end to end,
// inside the reference.
//
// INTEGRATION.md section 1 shows the change a gwgrid maintainer would make in
// run_grid's compute phase (proj/src/grid.cpp:519-558).  This program IS that
// change, compiled against the reference's own headers and linked with its
// own objects (oracle/refbuild/Makefile; Eigen stand-in) and with the engine's
// C ABI (include/gwgrid_cuda.h): the reference's generator, GWG1 streams,
// TileParams, ResultTile and result writer on both sides, and
//   * CPU side: the reference's preloop_stream_transform + run_grid (CT),
//   * device side: the same traversal with load_pass -> gwg_set_traits and
//     compute_tile -> gwg_solve_snp_slab straight into the reference's
//     ResultTile (GWG_LAYOUT_STREAM, ldo = rows), written by the reference's
//     OutputStream::write_result_cells.
// It then reads both result streams with the reference's reader and prints the
// reference's verify metric (norm-wise relative error per cell) and whether an
// injected zero variant column raises NotPositiveDefiniteError with the same
// (snp, trait) on both sides.  Run on the GPU box by
// tests/test_gpu_ref_golden.py::test_dropin_inside_reference_run_grid.
//
// usage: dropin_run_grid <workdir> [n p m t mb tb seed real|codes]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <vector>

#include "gwgrid/datagen.hpp"
#include "gwgrid/grid.hpp"
#include "gwgrid/stream.hpp"
#include "gwgrid/types.hpp"
#include "gwgrid_cuda.h"

namespace fs = std::filesystem;
using namespace gwgrid;

namespace {

void throw_if(const gwg_status& st) {  // INTEGRATION.md section 1, types.hpp:34-94
  if (st.code == GWG_OK) return;
  if (st.code == GWG_NOT_POSITIVE_DEFINITE)
    throw NotPositiveDefiniteError(st.msg, st.snp_index, st.trait_index);
  if (st.code == GWG_DIMENSION) throw DimensionError(st.msg);
  throw BackendError(st.msg);
}

void write_snps(const fs::path& path, const Eigen::MatrixXd& snps) {
  StreamHeader h;
  h.kind = StreamKind::snp;
  h.dims = {static_cast<std::uint64_t>(snps.rows()), static_cast<std::uint64_t>(snps.cols()), 0};
  OutputStream out = OutputStream::create(path, h);
  out.write_columns(0, snps.cols(), snps.data());
  out.finalize();
}

void write_traits(const fs::path& path, const Dataset& ds) {
  StreamHeader h;
  h.kind = StreamKind::trait;
  h.dims = {static_cast<std::uint64_t>(ds.traits.rows()),
            static_cast<std::uint64_t>(ds.traits.cols()), 0};
  OutputStream out = OutputStream::create(path, h);
  out.write_columns(0, ds.traits.cols(), ds.traits.data());
  out.write_trait_scalars(ds.h2.data(), ds.sigma2.data());
  out.finalize();
}

// run_grid's CT traversal (grid.cpp:495-556) with the device at the two seams.
void run_grid_device(const GridPrecompute& pre, const Eigen::MatrixXd& xl,
                     const fs::path& snps_rot_path, const fs::path& traits_path,
                     const fs::path& out_path, const TileParams& params, bool codes) {
  const InputStream snps = InputStream::open(snps_rot_path, StreamKind::snp);
  const InputStream traits = InputStream::open(traits_path, StreamKind::trait);
  const std::int64_t n = pre.n(), p = pre.p(), m = snps.count(), t = traits.count();

  gwg_status st{};
  gwg_engine* eng = gwg_engine_create(/*device=*/0, n, p, &st);
  if (!eng) throw_if(st);
  try {
    gwg_set_spectrum(eng, pre.spectrum.basis.data(), pre.spectrum.values.data(), GWG_HOST, &st);
    throw_if(st);
    gwg_set_covariates(eng, xl.data(), GWG_HOST, &st);  // raw X_L; rotated on device
    throw_if(st);
    // rotated slabs are real-valued: the FP64 path; raw genotype codes may use
    // the exact int8 path (then the raw stream is passed, is_rotated = 0)
    gwg_set_snp_coding(eng, codes ? GWG_SNP_GENOTYPES : GWG_SNP_REAL, &st);
    throw_if(st);

    StreamHeader h;
    h.kind = StreamKind::result;
    h.dims = {static_cast<std::uint64_t>(m), static_cast<std::uint64_t>(t),
              static_cast<std::uint64_t>(p)};
    OutputStream out = OutputStream::create(out_path, h);

    Eigen::MatrixXd trait_slab(n, params.tb), slab(n, params.mb);
    std::vector<double> h2(static_cast<std::size_t>(params.tb)), s2(h2.size());
    ResultTile tile;
    for (std::int64_t j0 = 0; j0 < t; j0 += params.tb) {
      const std::int64_t cols = std::min(params.tb, t - j0);
      // load_pass: replaces transform_trait_slab + build_trait_contexts
      traits.read_columns(j0, cols, trait_slab.data());
      traits.read_scalars(j0, cols, h2.data(), s2.data());
      gwg_set_traits(eng, cols, trait_slab.data(), h2.data(), s2.data(), GWG_HOST,
                     /*is_rotated=*/0, &st);
      throw_if(st);
      gwg_synchronize(eng, &st);  // weight-floor failures (-1, j) surface here
      if (st.code == GWG_NOT_POSITIVE_DEFINITE && st.trait_index >= 0) st.trait_index += j0;
      throw_if(st);
      for (std::int64_t i0 = 0; i0 < m; i0 += params.mb) {
        const std::int64_t rows = std::min(params.mb, m - i0);
        snps.read_columns(i0, rows, slab.data());
        tile.reset(i0, j0, rows, cols, p);
        // compute step: replaces compute_tile(contexts, slab.leftCols(rows), ...)
        gwg_solve_snp_slab(eng, i0, rows, slab.data(), GWG_HOST, /*is_rotated=*/codes ? 0 : 1,
                           tile.data.data(), GWG_HOST, GWG_LAYOUT_STREAM, /*ldo=*/rows, &st);
        if (st.code == GWG_NOT_POSITIVE_DEFINITE && st.trait_index >= 0) st.trait_index += j0;
        throw_if(st);
        out.write_result_cells(tile.i0, tile.j0, tile.rows, tile.cols, tile.data.data());
      }
    }
    out.finalize();
  } catch (...) {
    gwg_engine_destroy(eng);
    throw;
  }
  gwg_engine_destroy(eng);
}

double max_normwise(const fs::path& a_path, const fs::path& b_path) {
  const InputStream a = InputStream::open(a_path, StreamKind::result);
  const InputStream b = InputStream::open(b_path, StreamKind::result);
  if (a.rows() != b.rows() || a.count() != b.count() || a.coeffs() != b.coeffs()) return INFINITY;
  const std::int64_t p = a.coeffs();
  std::vector<double> ca(static_cast<std::size_t>(p)), cb(ca.size());
  double worst = 0.0;
  for (std::int64_t j = 0; j < a.count(); ++j)
    for (std::int64_t i = 0; i < a.rows(); ++i) {
      a.read_result_cell(i, j, ca.data());
      b.read_result_cell(i, j, cb.data());
      double num = 0.0, den = 0.0;
      for (std::int64_t c = 0; c < p; ++c) {
        num += (ca[c] - cb[c]) * (ca[c] - cb[c]);
        den += cb[c] * cb[c];
      }
      const double rel = std::sqrt(num) / std::sqrt(den);
      if (!(rel <= worst)) worst = rel;  // NaN propagates
    }
  return worst;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <workdir> [n p m t mb tb seed real|codes]\n", argv[0]);
    return 2;
  }
  const fs::path dir(argv[1]);
  auto arg = [&](int k, std::int64_t dflt) { return argc > k ? std::atoll(argv[k]) : dflt; };
  GenSpec spec;
  spec.dims.n = arg(2, 96);
  spec.dims.p = arg(3, 4);
  spec.dims.m = arg(4, 300);
  spec.dims.t = arg(5, 50);
  const std::int64_t mb = arg(6, 128), tb = arg(7, 20);
  spec.seed = static_cast<std::uint64_t>(arg(8, 7));
  const bool codes = argc > 9 && std::string(argv[9]) == "codes";
  try {
    fs::create_directories(dir);
    Dataset ds = generate_in_memory(spec);  // the reference's own generator
    if (codes) {  // genotype codes {0, 1, 2} from the reference's normal draws
      for (std::int64_t j = 0; j < ds.snps.cols(); ++j)
        for (std::int64_t i = 0; i < ds.snps.rows(); ++i)
          ds.snps(i, j) = ds.snps(i, j) < -0.5 ? 0.0 : ds.snps(i, j) < 0.8 ? 1.0 : 2.0;
    }
    const fs::path snps = dir / "snps.gwg", rot = dir / "snps_rot.gwg", traits = dir / "traits.gwg";
    const fs::path out_cpu = dir / "b_cpu.gwg", out_dev = dir / "b_dev.gwg";
    write_snps(snps, ds.snps);
    write_traits(traits, ds);

    RunCounters counters;
    const GridPrecompute pre = precompute_grid(ds.kinship, ds.xl, counters);
    RunOptions options;
    TileParams flags;
    flags.mb = mb;
    flags.tb = tb;
    options.params = flags.resolved(spec.dims);
    options.workers = 2;
    preloop_stream_transform(pre, snps, rot, options.params.nb, true, counters);
    run_grid(pre, rot, traits, out_cpu, options, counters);                          // reference
    run_grid_device(pre, ds.xl, codes ? snps : rot, traits, out_dev, options.params, codes);  // device
    const double err = max_normwise(out_dev, out_cpu);
    std::printf("cells=%lld max_normwise_rel_err=%.3e\n",
                static_cast<long long>(spec.dims.m * spec.dims.t), err);

    // identical failure: a zero variant column is not positive definite
    const std::int64_t bad = spec.dims.m / 2;
    for (std::int64_t i = 0; i < ds.snps.rows(); ++i) ds.snps(i, bad) = 0.0;
    write_snps(snps, ds.snps);
    preloop_stream_transform(pre, snps, rot, options.params.nb, true, counters);
    long long cpu_i = -2, cpu_j = -2, dev_i = -2, dev_j = -2;
    try {
      run_grid(pre, rot, traits, out_cpu, options, counters);
    } catch (const NotPositiveDefiniteError& e) {
      cpu_i = e.snp_index, cpu_j = e.trait_index;
    }
    try {
      run_grid_device(pre, ds.xl, codes ? snps : rot, traits, out_dev, options.params, codes);
    } catch (const NotPositiveDefiniteError& e) {
      dev_i = e.snp_index, dev_j = e.trait_index;
    }
    bool unreadable = false;
    try {
      InputStream::open(out_dev, StreamKind::result);
    } catch (const IncompleteStreamError&) {
      unreadable = true;
    }
    std::printf("npd_cpu=(%lld,%lld) npd_device=(%lld,%lld) failed_output_unreadable=%d\n", cpu_i,
                cpu_j, dev_i, dev_j, unreadable ? 1 : 0);
    // (which failing trait is reported first depends on the CPU pool's block order)
    const bool ok = err <= 1e-10 && cpu_i == bad && dev_i == bad && cpu_j >= 0 &&
                    cpu_j < spec.dims.t && dev_j >= 0 && dev_j < spec.dims.t && unreadable;
    std::printf("status=%s\n", ok ? "ok" : "FAILED");
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("status=error what=%s\n", e.what());
    return 3;
  }
}
