// gwgrid_cuda.hpp — header-only C++ host mirror of the reference gwgrid API
// over the C ABI in gwgrid_cuda.h.
//
// Same names, argument meaning and error behaviour as the reference's C++
// library for the hot path (proj/include/gwgrid/grid.hpp, gls.hpp,
// types.hpp), so a caller of gwgrid's compute_tile / run_grid switches by
// changing the namespace:
//
//   gwgrid::DimensionError / NotPositiveDefiniteError{snp_index, trait_index}
//   / BackendError / InfeasibleBudgetError / IoError      (types.hpp:34-94)
//   DeviceGrid::precompute(...)      <- precompute_grid           (grid.hpp:81-101)
//   DeviceGrid::build_trait_contexts <- build_trait_contexts      (grid.hpp:121-125)
//   DeviceGrid::compute_tile(...)    <- compute_tile + ResultTile (grid.hpp:129-169)
//   DeviceGrid::run_grid(...)        <- run_grid (in-memory)      (grid.hpp:212-237)
//
// Matrices are plain column-major double buffers (the layout of the
// reference's Eigen::MatrixXd), passed as pointer + dims.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gwgrid_cuda.h"

namespace gwgrid_cuda {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct NonSymmetricError : Error {
  using Error::Error;
};
struct BackendError : Error {
  using Error::Error;
};
struct NotPositiveDefiniteError : Error {
  std::int64_t snp_index = -1;
  std::int64_t trait_index = -1;
  NotPositiveDefiniteError(const std::string& msg, std::int64_t snp, std::int64_t trait)
      : Error(msg), snp_index(snp), trait_index(trait) {}
};
struct IoError : Error {
  using Error::Error;
};
struct InfeasibleBudgetError : Error {
  using Error::Error;
};
struct DeviceError : Error {
  using Error::Error;
};

inline void throw_if(const gwg_status& st) {
  switch (st.code) {
    case GWG_OK:
      return;
    case GWG_DIMENSION:
      throw DimensionError(st.msg);
    case GWG_NON_SYMMETRIC:
      throw NonSymmetricError(st.msg);
    case GWG_BACKEND:
      throw BackendError(st.msg);
    case GWG_NOT_POSITIVE_DEFINITE:
      throw NotPositiveDefiniteError(st.msg, st.snp_index, st.trait_index);
    case GWG_IO:
      throw IoError(st.msg);
    case GWG_INFEASIBLE_BUDGET:
      throw InfeasibleBudgetError(st.msg);
    default:
      throw DeviceError(st.msg);
  }
}

// ResultTile (grid.hpp:129-148): coefficient-fastest, then local SNP row,
// then local trait column: data[(jl * rows + il) * p + c].
struct ResultTile {
  std::int64_t i0 = 0, j0 = 0, rows = 0, cols = 0, p = 0;
  std::vector<double> data;
  void reset(std::int64_t i0_, std::int64_t j0_, std::int64_t rows_, std::int64_t cols_,
             std::int64_t p_) {
    i0 = i0_;
    j0 = j0_;
    rows = rows_;
    cols = cols_;
    p = p_;
    data.resize(static_cast<std::size_t>(rows_ * cols_ * p_));
  }
  double* cell(std::int64_t il, std::int64_t jl) { return data.data() + (jl * rows + il) * p; }
  const double* cell(std::int64_t il, std::int64_t jl) const {
    return data.data() + (jl * rows + il) * p;
  }
};

// One device engine (one per GPU; calls serialised by the caller).
class DeviceGrid {
 public:
  DeviceGrid(int device, std::int64_t n, std::int64_t p) : n_(n), p_(p) {
    gwg_status st{};
    e_ = gwg_engine_create(device, n, p, &st);
    if (!e_) throw_if(st);
  }
  ~DeviceGrid() { gwg_engine_destroy(e_); }
  DeviceGrid(const DeviceGrid&) = delete;
  DeviceGrid& operator=(const DeviceGrid&) = delete;

  std::int64_t n() const { return n_; }
  std::int64_t p() const { return p_; }

  // precompute_grid with the eigensystem computed by the caller on the CPU
  // (eigendecompose_kinship stays on the host): basis n x n, ascending values,
  // raw covariates n x (p-1).
  void precompute(const double* basis, const double* values, const double* xl) {
    gwg_status st{};
    gwg_set_spectrum(e_, basis, values, GWG_HOST, &st);
    throw_if(st);
    gwg_set_covariates(e_, xl, GWG_HOST, &st);
    throw_if(st);
  }

  // Integer genotype codes in every SNP slab from now on (GWG_SNP_GENOTYPES:
  // exact int8 tensor-core rotation + split grid) or real values (default).
  void set_snp_coding(int coding) {
    gwg_status st{};
    gwg_set_snp_coding(e_, coding, &st);
    throw_if(st);
  }

  // transform_trait_slab + build_trait_contexts for a raw trait slab n x t
  // (trait0 only tags errors in the reference; traits are 0-based here).
  // Like the reference (grid.cpp:146-175) this throws a trait's weight-floor
  // failure here: the asynchronous gwg_set_traits is followed by one
  // gwg_synchronize, which reports it.
  void build_trait_contexts(const double* traits, std::int64_t t, const double* h2,
                            const double* sigma2, bool rotated = false) {
    gwg_status st{};
    gwg_set_traits(e_, t, traits, h2, sigma2, GWG_HOST, rotated ? 1 : 0, &st);
    throw_if(st);
    gwg_synchronize(e_, &st);
    throw_if(st);
    t_ = t;
  }

  // compute_tile: every cell of `tile` (rows SNP columns at global i0 x all
  // installed traits) from an n x rows SNP slab, raw unless `rotated`.
  void compute_tile(const double* snp_slab, ResultTile& tile, bool rotated = false) {
    if (tile.cols != t_ || tile.p != p_) throw DimensionError("tile shape disagrees with traits");
    gwg_status st{};
    gwg_solve_snp_slab(e_, tile.i0, tile.rows, snp_slab, GWG_HOST, rotated ? 1 : 0,
                       tile.data.data(), GWG_HOST, GWG_LAYOUT_STREAM, tile.rows, &st);
    throw_if(st);
  }

  // run_grid over an in-memory raw SNP matrix n x m; b is (j*m + i)*p
  // (result stream order) or (i*t + j)*p with numpy_layout.
  gwg_counters run_grid(const double* snps, std::int64_t m, double* b,
                        bool numpy_layout = false, std::int64_t mb = 0) {
    gwg_status st{};
    gwg_run_options o{mb, numpy_layout ? GWG_LAYOUT_NUMPY : GWG_LAYOUT_STREAM, 1};
    gwg_counters c{};
    gwg_run_grid(e_, m, snps, b, &o, &c, &st);
    throw_if(st);
    return c;
  }

 private:
  gwg_engine* e_ = nullptr;
  std::int64_t n_, p_, t_ = 0;
};

}  // namespace gwgrid_cuda
