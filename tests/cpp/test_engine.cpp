// C++ parity tests for the host mirror (include/gwgrid_cuda.hpp) — written
// like the reference's doctest suites (proj/tests/test_grid.cpp), checking the
// device engine against the oracle's C++ restatement (oracle/gls_oracle.cpp,
// test infrastructure).  Needs a B200; run by tests/test_cpp.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "gwgrid_cuda.hpp"

extern "C" {
struct orc_status {
  int code;
  int64_t snp_index, trait_index;
  char msg[256];
};
int orc_eigendecompose(int64_t, const double*, double*, double*, orc_status*);
int orc_rotate(int64_t, const double*, int64_t, const double*, double*);
int orc_compute_grid(int64_t, int64_t, int64_t, int64_t, const double*, const double*,
                     const double*, const double*, const double*, const double*, int64_t,
                     int64_t, int, int, double*, orc_status*);
}

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                           \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(cond)) {                                                            \
      ++g_fail;                                                               \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
    }                                                                         \
  } while (0)

struct Data {
  int64_t n, p, m, t;
  std::vector<double> phi, basis, values, xl, snps, traits, h2, sigma2;
  Data(int64_t n_, int64_t p_, int64_t m_, int64_t t_, uint64_t seed)
      : n(n_), p(p_), m(m_), t(t_) {
    std::vector<double> g(n * 2 * n);
    gwg_gen_genotypes(seed, 1, n, 0, 2 * n, 1, g.data(), n);
    phi.assign(n * n, 0.0);
    for (int64_t a = 0; a < n; ++a)
      for (int64_t b = 0; b <= a; ++b) {
        double s = 0;
        for (int64_t k = 0; k < 2 * n; ++k) s += g[a + k * n] * g[b + k * n];
        phi[a + b * n] = phi[b + a * n] = s / double(2 * n) + (a == b ? 1e-3 : 0.0);
      }
    basis.resize(n * n);
    values.resize(n);
    orc_status st{};
    orc_eigendecompose(n, phi.data(), basis.data(), values.data(), &st);
    xl.resize(n * (p - 1));
    for (int64_t i = 0; i < n && p > 1; ++i) xl[i] = 1.0;
    if (p > 2) gwg_gen_normals(seed, 2, n, 0, p - 2, xl.data() + n, n);
    snps.resize(n * m);
    gwg_gen_genotypes(seed, 3, n, 0, m, 0, snps.data(), n);
    traits.resize(n * t);
    gwg_gen_normals(seed, 4, n, 0, t, traits.data(), n);
    h2.resize(t);
    gwg_gen_uniform(seed, 5, t, 0.05, 0.95, h2.data());
    sigma2.assign(t, 1.0);
  }
  // oracle result in ResultTile order (j*m + i)*p
  std::vector<double> oracle() const {
    std::vector<double> xlr(n * (p - 1) + 1), xr(n * m), yr(n * t), out(m * t * p);
    if (p > 1) orc_rotate(n, basis.data(), p - 1, xl.data(), xlr.data());
    orc_rotate(n, basis.data(), m, snps.data(), xr.data());
    orc_rotate(n, basis.data(), t, traits.data(), yr.data());
    orc_status st{};
    orc_compute_grid(n, p, m, t, values.data(), xlr.data(), xr.data(), yr.data(), h2.data(),
                     sigma2.data(), 0, 0, 4, 1, out.data(), &st);
    return out;
  }
};

static double max_normwise(const std::vector<double>& a, const std::vector<double>& b,
                           int64_t p) {
  double worst = 0;
  for (size_t c = 0; c < a.size() / p; ++c) {
    double d = 0, r = 0;
    for (int64_t q = 0; q < p; ++q) {
      d += (a[c * p + q] - b[c * p + q]) * (a[c * p + q] - b[c * p + q]);
      r += b[c * p + q] * b[c * p + q];
    }
    worst = std::max(worst, std::sqrt(d / r));
  }
  return worst;
}

static void test_compute_tile_matches_oracle() {
  Data d(200, 4, 150, 37, 5);
  gwgrid_cuda::DeviceGrid grid(0, d.n, d.p);
  grid.precompute(d.basis.data(), d.values.data(), d.xl.data());
  grid.build_trait_contexts(d.traits.data(), d.t, d.h2.data(), d.sigma2.data());
  gwgrid_cuda::ResultTile tile;
  tile.reset(0, 0, d.m, d.t, d.p);
  grid.compute_tile(d.snps.data(), tile);
  const double err = max_normwise(tile.data, d.oracle(), d.p);
  std::printf("  compute_tile vs oracle: max norm-wise rel err %.3e\n", err);
  CHECK(err < 1e-12);
  // run_grid (stream order) is bitwise identical to compute_tile
  std::vector<double> b(d.m * d.t * d.p);
  grid.run_grid(d.snps.data(), d.m, b.data(), false, 64);
  CHECK(std::memcmp(b.data(), tile.data.data(), b.size() * sizeof(double)) == 0);
}

static void test_genotype_coding_matches_oracle() {
  Data d(200, 4, 150, 37, 5);  // the generator's SNPs are genotype codes {0,1,2}
  gwgrid_cuda::DeviceGrid grid(0, d.n, d.p);
  grid.precompute(d.basis.data(), d.values.data(), d.xl.data());
  grid.set_snp_coding(GWG_SNP_GENOTYPES);
  grid.build_trait_contexts(d.traits.data(), d.t, d.h2.data(), d.sigma2.data());
  gwgrid_cuda::ResultTile tile;
  tile.reset(0, 0, d.m, d.t, d.p);
  grid.compute_tile(d.snps.data(), tile);
  const double err = max_normwise(tile.data, d.oracle(), d.p);
  std::printf("  genotype compute_tile vs oracle: max norm-wise rel err %.3e\n", err);
  CHECK(err < 1e-12);
  std::vector<double> b(d.m * d.t * d.p);
  grid.run_grid(d.snps.data(), d.m, b.data(), false, 64);
  CHECK(std::memcmp(b.data(), tile.data.data(), b.size() * sizeof(double)) == 0);
}

static void test_zero_column_npd_coordinates() {
  Data d(48, 3, 12, 6, 4);
  for (int64_t k = 0; k < d.n; ++k) d.snps[5 * d.n + k] = 0.0;
  gwgrid_cuda::DeviceGrid grid(0, d.n, d.p);
  grid.precompute(d.basis.data(), d.values.data(), d.xl.data());
  grid.build_trait_contexts(d.traits.data(), d.t, d.h2.data(), d.sigma2.data());
  gwgrid_cuda::ResultTile tile;
  tile.reset(0, 0, d.m, d.t, d.p);
  bool threw = false;
  try {
    grid.compute_tile(d.snps.data(), tile);
  } catch (const gwgrid_cuda::NotPositiveDefiniteError& e) {
    threw = true;
    CHECK(e.snp_index == 5);
    CHECK(e.trait_index == 0);
  }
  CHECK(threw);
}

static void test_trait_weight_failure() {
  const int64_t n = 8;
  std::vector<double> basis(n * n, 0.0), values(n), xl(n, 1.0), y(n * 5), h2(5, 0.0), s2(5, 1.0);
  for (int64_t i = 0; i < n; ++i) {
    basis[i + i * n] = 1.0;
    values[i] = double(i) - 0.5;
  }
  gwg_gen_normals(3, 4, n, 0, 5, y.data(), n);
  h2[3] = 0.9;
  gwgrid_cuda::DeviceGrid grid(0, n, 2);
  grid.precompute(basis.data(), values.data(), xl.data());
  bool threw = false;
  try {
    grid.build_trait_contexts(y.data(), 5, h2.data(), s2.data());
  } catch (const gwgrid_cuda::NotPositiveDefiniteError& e) {
    threw = true;
    CHECK(e.snp_index == -1);
    CHECK(e.trait_index == 3);
  }
  CHECK(threw);
}

static void test_dimension_errors() {
  bool threw = false;
  try {
    gwgrid_cuda::DeviceGrid bad(0, 4, 5);
  } catch (const gwgrid_cuda::DimensionError&) {
    threw = true;
  }
  CHECK(threw);
}

int main() {
  const std::pair<const char*, std::function<void()>> cases[] = {
      {"compute_tile matches the oracle; run_grid bitwise equal", test_compute_tile_matches_oracle},
      {"genotype coding (int8 tensor-core path) matches the oracle",
       test_genotype_coding_matches_oracle},
      {"zero variant column fails with coordinates", test_zero_column_npd_coordinates},
      {"trait weight failure surfaces the trait index", test_trait_weight_failure},
      {"dimension errors", test_dimension_errors},
  };
  for (const auto& c : cases) {
    std::printf("[case] %s\n", c.first);
    try {
      c.second();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  unexpected exception: %s\n", e.what());
    }
  }
  std::printf("[summary] %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
