// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.  A thin C face over the REFERENCE's
// own compiled sources (gwgrid: gls.cpp, grid.cpp, stream.cpp, pool.cpp,
// pipeline.cpp, types.cpp, compiled where they lie under /root/reference by
// oracle/refbuild/Makefile against the Eigen stand-in header) so that Python
// can run the reference here, pin oracle/gls_oracle.cpp against it and write
// the golden vectors under tests/golden/ (tests/golden/make_ref_golden.py).
// Nothing in this file computes: every number comes from a gwgrid:: call.
//
// ref_solve_grid follows python/bindings.cpp:115-190 (solve_grid_py): stage
// GWG1 files, precompute_grid, preloop_stream_transform, run_grid /
// run_grid_naive, read the result stream back cell by cell.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <optional>
#include <string>
#include <vector>

#include "gwgrid/datagen.hpp"
#include "gwgrid/gls.hpp"
#include "gwgrid/grid.hpp"
#include "gwgrid/pool.hpp"
#include "gwgrid/stream.hpp"
#include "gwgrid/types.hpp"

namespace fs = std::filesystem;
using namespace gwgrid;

extern "C" {

struct ref_status {
  std::int32_t code;  // 0 ok, 1 dimension, 2 non-symmetric, 3 backend, 4 not positive definite,
                      // 5 io/stream, 6 other gwgrid::Error, 7 anything else
  std::int64_t snp_index;
  std::int64_t trait_index;
  char msg[256];
};

}  // extern "C"

namespace {

void set_msg(ref_status* st, int code, const char* what, std::int64_t i = -1, std::int64_t j = -1) {
  if (!st) return;
  st->code = code;
  st->snp_index = i;
  st->trait_index = j;
  std::snprintf(st->msg, sizeof st->msg, "%s", what);
}

template <class F>
int guarded(ref_status* st, F&& f) {
  set_msg(st, 0, "");
  try {
    f();
    return 0;
  } catch (const NotPositiveDefiniteError& e) {
    set_msg(st, 4, e.what(), e.snp_index, e.trait_index);
  } catch (const DimensionError& e) {
    set_msg(st, 1, e.what());
  } catch (const NonSymmetricError& e) {
    set_msg(st, 2, e.what());
  } catch (const BackendError& e) {
    set_msg(st, 3, e.what());
  } catch (const IoError& e) {
    set_msg(st, 5, e.what());
  } catch (const Error& e) {
    set_msg(st, 6, e.what());
  } catch (const std::exception& e) {
    set_msg(st, 7, e.what());
  }
  return st ? st->code : -1;
}

Eigen::MatrixXd mat(const double* p, std::int64_t r, std::int64_t c) {
  Eigen::MatrixXd m(r, c);
  if (r * c > 0) std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(r * c));
  return m;
}
Eigen::VectorXd vec(const double* p, std::int64_t n) {
  Eigen::VectorXd v(n);
  if (n > 0) std::memcpy(v.data(), p, sizeof(double) * static_cast<std::size_t>(n));
  return v;
}
void put(const Eigen::MatrixXd& m, double* dst) {
  if (m.size() > 0) std::memcpy(dst, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
}
void put(const Eigen::VectorXd& v, double* dst) {
  if (v.size() > 0) std::memcpy(dst, v.data(), sizeof(double) * static_cast<std::size_t>(v.size()));
}

KinshipSpectrum spectrum_of(std::int64_t n, const double* basis, const double* values) {
  KinshipSpectrum s;
  s.basis = mat(basis, n, n);
  s.values = vec(values, n);
  return s;
}

void stage_snps(const fs::path& path, const double* snps, std::int64_t n, std::int64_t m) {
  StreamHeader h;
  h.kind = StreamKind::snp;
  h.dims = {static_cast<std::uint64_t>(n), static_cast<std::uint64_t>(m), 0};
  OutputStream out = OutputStream::create(path, h);
  out.write_columns(0, m, snps);
  out.finalize();
}
void stage_traits(const fs::path& path, const double* traits, const double* h2, const double* s2,
                  std::int64_t n, std::int64_t t) {
  StreamHeader h;
  h.kind = StreamKind::trait;
  h.dims = {static_cast<std::uint64_t>(n), static_cast<std::uint64_t>(t), 0};
  OutputStream out = OutputStream::create(path, h);
  out.write_columns(0, t, traits);
  out.write_trait_scalars(h2, s2);
  out.finalize();
}

// run_grid / run_grid_naive over staged files, as bindings.cpp:143-166.
void run_files(const Eigen::MatrixXd& kinship, const Eigen::MatrixXd& xl, const fs::path& snps_path,
               const fs::path& traits_path, const fs::path& rotated_path, const fs::path& out_path,
               int scheduler, int workers, std::int64_t nb, std::int64_t mb, std::int64_t tb,
               std::int64_t mbb, std::int64_t tbb, int double_buffer, std::uint64_t* counters_out) {
  RunCounters counters;
  const GridPrecompute pre = precompute_grid(kinship, xl, counters);
  if (scheduler == 2) {
    run_grid_naive(pre, snps_path, traits_path, out_path, counters);
  } else {
    const InputStream probe_s = InputStream::open(snps_path, StreamKind::snp);
    const InputStream probe_t = InputStream::open(traits_path, StreamKind::trait);
    ProblemDims dims;
    dims.n = kinship.rows();
    dims.p = xl.cols() + 1;
    dims.m = probe_s.count();
    dims.t = probe_t.count();
    RunOptions options;
    TileParams flags{nb, mb, tb, mbb, tbb};
    options.scheduler = scheduler == 1 ? Scheduler::it : Scheduler::ct;
    options.workers = workers;
    options.double_buffer = double_buffer != 0;
    options.params = flags.resolved(dims);
    preloop_stream_transform(pre, snps_path, rotated_path, options.params.nb, double_buffer != 0,
                             counters);
    run_grid(pre, rotated_path, traits_path, out_path, options, counters);
  }
  if (counters_out) {
    const FlopIoCounters snap = counters.snapshot();
    counters_out[0] = snap.bytes_loaded;
    counters_out[1] = snap.bytes_stored;
    counters_out[2] = snap.context_builds;
  }
}

}  // namespace

extern "C" {

int ref_eigendecompose(std::int64_t n, const double* phi, double* basis, double* values,
                       ref_status* st) {
  return guarded(st, [&] {
    const KinshipSpectrum s = eigendecompose_kinship(mat(phi, n, n));
    put(s.basis, basis);
    put(s.values, values);
  });
}

int ref_trait_weights(std::int64_t n, const double* values, double h2, double sigma2,
                      std::int64_t trait_index, double* d, double* k, ref_status* st) {
  return guarded(st, [&] {
    TraitScalars sc;
    sc.h2 = h2;
    sc.sigma2 = sigma2;
    const TraitWeights w = build_trait_weights(vec(values, n), sc, trait_index);
    put(w.d, d);
    put(w.k, k);
  });
}

int ref_trait_context(std::int64_t n, std::int64_t pm1, const double* values, const double* xl_rot,
                      const double* y_rot, double h2, double sigma2, std::int64_t trait_index,
                      double* v, double* w_l, double* s_tl, double* b_t, ref_status* st) {
  return guarded(st, [&] {
    TraitScalars sc;
    sc.h2 = h2;
    sc.sigma2 = sigma2;
    const Eigen::MatrixXd xl = mat(xl_rot, n, pm1);
    const Eigen::VectorXd y = vec(y_rot, n);
    const TraitContext ctx = build_trait_context(vec(values, n), xl, y, sc, trait_index);
    put(ctx.v, v);
    put(ctx.w_l, w_l);
    put(ctx.s_tl, s_tl);
    put(ctx.b_t, b_t);
  });
}

int ref_solve_partitioned(std::int64_t n, std::int64_t pm1, const double* basis,
                          const double* values, const double* xl, const double* xr,
                          const double* y, double h2, double sigma2, double* out, ref_status* st) {
  return guarded(st, [&] {
    TraitScalars sc;
    sc.h2 = h2;
    sc.sigma2 = sigma2;
    put(solve_partitioned_gls(spectrum_of(n, basis, values), mat(xl, n, pm1), vec(xr, n),
                              vec(y, n), sc),
        out);
  });
}

int ref_solve_single(std::int64_t n, std::int64_t p, const double* basis, const double* values,
                     const double* x, const double* y, double h2, double sigma2, double* out,
                     ref_status* st) {
  return guarded(st, [&] {
    TraitScalars sc;
    sc.h2 = h2;
    sc.sigma2 = sigma2;
    put(solve_single_gls(spectrum_of(n, basis, values), mat(x, n, p), vec(y, n), sc), out);
  });
}

// The reference's independent dense-Cholesky route (gls.cpp:188-244) for a
// list of cells of one problem: cells[k] = (i, j).
int ref_cholesky_cells(std::int64_t n, std::int64_t pm1, std::int64_t m, std::int64_t t,
                       const double* phi, const double* xl, const double* snps,
                       const double* traits, const double* h2, const double* sigma2,
                       std::int64_t n_cells, const std::int64_t* cells, double* out,
                       ref_status* st) {
  return guarded(st, [&] {
    (void)m;
    (void)t;
    const CholeskyOracle oracle(mat(phi, n, n));
    const Eigen::MatrixXd xlm = mat(xl, n, pm1);
    std::int64_t cached_j = -1;
    std::optional<CholeskyOracle::TraitFactor> factor;
    for (std::int64_t c = 0; c < n_cells; ++c) {
      const std::int64_t i = cells[2 * c], j = cells[2 * c + 1];
      if (j != cached_j) {
        TraitScalars sc;
        sc.h2 = h2[j];
        sc.sigma2 = sigma2[j];
        factor.emplace(oracle.factor(sc, j));
        cached_j = j;
      }
      const Eigen::VectorXd b =
          factor->solve(xlm, vec(snps + i * n, n), vec(traits + j * n, n));
      put(b, out + c * (pm1 + 1));
    }
  });
}

// In-memory operands staged to GWG1 files under workdir by the reference's
// own writer, solved by the reference's streamed engine, read back by its
// reader.  b is (m, t, p) C-contiguous like gwgrid.solve_grid's result.
int ref_solve_grid(std::int64_t n, std::int64_t p, std::int64_t m, std::int64_t t,
                   const double* kinship, const double* xl, const double* snps,
                   const double* traits, const double* h2, const double* sigma2, int scheduler,
                   int workers, std::int64_t nb, std::int64_t mb, std::int64_t tb,
                   std::int64_t mbb, std::int64_t tbb, int double_buffer, const char* workdir,
                   double* b, std::uint64_t* counters_out, ref_status* st) {
  return guarded(st, [&] {
    const fs::path dir(workdir);
    const fs::path snps_path = dir / "snps.gwg", traits_path = dir / "traits.gwg";
    const fs::path out_path = dir / "b.gwg", rotated = dir / "snps_rot.gwg";
    stage_snps(snps_path, snps, n, m);
    stage_traits(traits_path, traits, h2, sigma2, n, t);
    run_files(mat(kinship, n, n), mat(xl, n, p - 1), snps_path, traits_path, rotated, out_path,
              scheduler, workers, nb, mb, tb, mbb, tbb, double_buffer, counters_out);
    const InputStream results = InputStream::open(out_path, StreamKind::result);
    for (std::int64_t j = 0; j < t; ++j)
      for (std::int64_t i = 0; i < m; ++i)
        results.read_result_cell(i, j, b + (static_cast<std::size_t>(i) * t + j) * p);
  });
}

// The same engine over GWG1 files somebody else wrote (our gwg1.py codec /
// our engine's file legs): pins the file format both ways.
int ref_run_grid_files(std::int64_t n, std::int64_t p, const double* kinship, const double* xl,
                       const char* snps_path, const char* traits_path, const char* rotated_path,
                       const char* out_path, int scheduler, int workers, std::int64_t nb,
                       std::int64_t mb, std::int64_t tb, std::int64_t mbb, std::int64_t tbb,
                       int double_buffer, std::uint64_t* counters_out, ref_status* st) {
  return guarded(st, [&] {
    run_files(mat(kinship, n, n), mat(xl, n, p - 1), snps_path, traits_path, rotated_path,
              out_path, scheduler, workers, nb, mb, tb, mbb, tbb, double_buffer, counters_out);
  });
}

// A result stream somebody else wrote (our engine's file leg), decoded by
// the reference's own reader (stream.cpp: header checks, completeness flag,
// positional cell reads) into (m, t, p) C order; dims[3] returns its header.
int ref_read_result(const char* path, std::int64_t* dims, double* b, std::int64_t capacity,
                    ref_status* st) {
  return guarded(st, [&] {
    const InputStream results = InputStream::open(path, StreamKind::result);
    const std::int64_t m = results.rows(), t = results.count(), p = results.coeffs();
    dims[0] = m;
    dims[1] = t;
    dims[2] = p;
    if (b == nullptr) return;
    if (capacity < m * t * p) throw DimensionError("result buffer too small");
    for (std::int64_t j = 0; j < t; ++j)
      for (std::int64_t i = 0; i < m; ++i)
        results.read_result_cell(i, j, b + (static_cast<std::size_t>(i) * t + j) * p);
  });
}

// The in-core traversal of run_grid (grid.cpp:495-556) without the file
// legs: rotate the covariates and the trait slab, build the contexts once,
// then per slab of mb variant columns transform_snp_slab + compute_tile (CT
// blocks on a WorkerPool).  Used as the timed CPU path of the reference
// build (bench.py --impl reference) and for in-memory pins.  b is (m, t, p).
int ref_compute_grid(std::int64_t n, std::int64_t p, std::int64_t m, std::int64_t t,
                     const double* basis, const double* values, const double* xl,
                     const double* snps, const double* traits, const double* h2,
                     const double* sigma2, int workers, std::int64_t mb, std::int64_t mbb,
                     std::int64_t tbb, double* b, ref_status* st) {
  return guarded(st, [&] {
    GridPrecompute pre;
    pre.spectrum = spectrum_of(n, basis, values);
    const Eigen::MatrixXd xlm = mat(xl, n, p - 1);
    pre.xl_rot.resize(n, p - 1);
    if (p > 1) rotate_columns(pre.spectrum.basis, xlm, pre.xl_rot);
    Eigen::MatrixXd trait_slab = mat(traits, n, t);
    transform_trait_slab(pre, trait_slab, nullptr);
    std::vector<TraitScalars> scalars(static_cast<std::size_t>(t));
    for (std::int64_t j = 0; j < t; ++j) {
      scalars[static_cast<std::size_t>(j)].h2 = h2[j];
      scalars[static_cast<std::size_t>(j)].sigma2 = sigma2[j];
    }
    const std::vector<TraitContext> contexts =
        build_trait_contexts(pre, trait_slab, scalars, 0, nullptr);
    ProblemDims dims;
    dims.n = n;
    dims.p = p;
    dims.m = m;
    dims.t = t;
    TileParams flags;
    flags.mb = mb;
    flags.mbb = mbb;
    flags.tbb = tbb;
    const TileParams params = flags.resolved(dims);
    WorkerPool pool(workers);
    Eigen::MatrixXd raw(n, params.mb), rot(n, params.mb);
    ResultTile tile;
    for (std::int64_t i0 = 0; i0 < m; i0 += params.mb) {
      const std::int64_t rows = std::min(params.mb, m - i0);
      std::memcpy(raw.data(), snps + i0 * n, sizeof(double) * static_cast<std::size_t>(rows * n));
      transform_snp_slab(pre, raw.leftCols(rows), rot.leftCols(rows), nullptr);
      tile.reset(i0, 0, rows, t, p);
      compute_tile(contexts, rot.leftCols(rows), params, tile, &pool, nullptr);
      for (std::int64_t jl = 0; jl < t; ++jl)
        for (std::int64_t il = 0; il < rows; ++il)
          std::memcpy(b + (static_cast<std::size_t>(i0 + il) * t + jl) * p, tile.cell(il, jl),
                      sizeof(double) * static_cast<std::size_t>(p));
    }
  });
}

// A gwgrid-dataset-1 directory written by the reference's own generator
// (datagen.cpp:263-315: manifest.txt + kinship / xl / snps / traits streams).
int ref_generate_dataset(const char* dir, std::int64_t n, std::int64_t p, std::int64_t m,
                         std::int64_t t, std::uint64_t seed, double condition, ref_status* st) {
  return guarded(st, [&] {
    GenSpec spec;
    spec.dims.n = n;
    spec.dims.p = p;
    spec.dims.m = m;
    spec.dims.t = t;
    spec.seed = seed;
    spec.condition = condition;
    generate_dataset(spec, dir);
  });
}

// A dataset directory somebody else wrote (our CLI's generate), parsed by the
// reference's load_manifest (datagen.cpp:317-396) and read by its stream
// reader: dims[4] = n, p, m, t from the manifest; sums[6] = plain sums of the
// kinship, xl, snps, traits, h2 and sigma2 payloads as the reference read them.
int ref_load_dataset(const char* manifest_path, std::int64_t* dims, double* sums, ref_status* st) {
  return guarded(st, [&] {
    const DatasetManifest man = load_manifest(manifest_path);
    dims[0] = man.spec.dims.n;
    dims[1] = man.spec.dims.p;
    dims[2] = man.spec.dims.m;
    dims[3] = man.spec.dims.t;
    sums[0] = read_dense(man.paths.kinship, StreamKind::operand).sum();
    sums[1] = man.spec.dims.p > 1 ? read_dense(man.paths.xl, StreamKind::operand).sum() : 0.0;
    sums[2] = read_dense(man.paths.snps, StreamKind::snp).sum();
    sums[3] = read_dense(man.paths.traits, StreamKind::trait).sum();
    const InputStream traits = InputStream::open(man.paths.traits, StreamKind::trait);
    std::vector<double> h2(static_cast<std::size_t>(traits.count())), s2(h2.size());
    traits.read_scalars(0, traits.count(), h2.data(), s2.data());
    sums[4] = sums[5] = 0.0;
    for (double v : h2) sums[4] += v;
    for (double v : s2) sums[5] += v;
  });
}

}  // extern "C"
