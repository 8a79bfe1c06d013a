// datagen.cpp — seeded synthetic inputs with BASELINE.json's generators.
//
// The reference's own generator (proj/src/datagen.cpp:82-182: mt19937_64 per
// component, random-SPD kinship, normal SNPs) does not match BASELINE.json's
// workload, so this is a fresh, counter-based one: every value is a pure
// function of (seed, matrix id, column, row), which lets any SNP range be
// generated on any rank or regenerated for a spot check without
// materialising the whole matrix.
//   column key   K = splitmix64(seed*phi64 + matrix*C1 + col)
//   element word w(K, idx) = splitmix64(K + idx*phi64)
//   uniform      u = (w >> 11) * 2^-53 in [0, 1)
//   genotype     g = [u(K,2r) < maf] + [u(K,2r+1) < maf],
//                maf = 0.05 + 0.45 u(splitmix64(K ^ C2), 0)   (Binomial(2, maf))
//   normal       Box-Muller on (1 - u(K,2r), u(K,2r+1))        (N(0,1))
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/gwgrid_cuda.h"

namespace {

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kC1 = 0xD1B54A32D192ED03ull;
constexpr uint64_t kC2 = 0xA5A5A5A5DEADBEEFull;

inline uint64_t splitmix64(uint64_t x) {
  x += kPhi;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

inline uint64_t col_key(uint64_t seed, int32_t matrix, int64_t col) {
  return splitmix64(seed * kPhi + uint64_t(matrix) * kC1 + uint64_t(col));
}

inline double u01(uint64_t key, uint64_t idx) {
  return double(splitmix64(key + idx * kPhi) >> 11) * 0x1.0p-53;
}

template <class F>
void parallel_cols(int64_t ncols, F&& f) {
  const int64_t work = ncols;
  unsigned hw = std::thread::hardware_concurrency();
  int threads = int(std::min<int64_t>(std::max(1u, hw), std::max<int64_t>(1, work / 16)));
  if (threads <= 1) {
    for (int64_t c = 0; c < ncols; ++c) f(c);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w)
    pool.emplace_back([&, w] {
      for (int64_t c = w; c < ncols; c += threads) f(c);
    });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

void gwg_gen_genotypes(uint64_t seed, int32_t matrix, int64_t rows, int64_t col0, int64_t ncols,
                       int32_t standardize, double* out, int64_t ld) {
  parallel_cols(ncols, [&](int64_t c) {
    const uint64_t key = col_key(seed, matrix, col0 + c);
    const double maf = 0.05 + 0.45 * u01(splitmix64(key ^ kC2), 0);
    const double mean = 2.0 * maf, sd = std::sqrt(2.0 * maf * (1.0 - maf));
    double* col = out + c * ld;
    for (int64_t r = 0; r < rows; ++r) {
      const double g = double(u01(key, 2 * uint64_t(r)) < maf) +
                       double(u01(key, 2 * uint64_t(r) + 1) < maf);
      col[r] = standardize ? (g - mean) / sd : g;
    }
  });
}

void gwg_gen_normals(uint64_t seed, int32_t matrix, int64_t rows, int64_t col0, int64_t ncols,
                     double* out, int64_t ld) {
  parallel_cols(ncols, [&](int64_t c) {
    const uint64_t key = col_key(seed, matrix, col0 + c);
    double* col = out + c * ld;
    for (int64_t r = 0; r < rows; ++r) {
      const double u1 = 1.0 - u01(key, 2 * uint64_t(r));
      const double u2 = u01(key, 2 * uint64_t(r) + 1);
      col[r] = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
  });
}

void gwg_gen_uniform(uint64_t seed, int32_t matrix, int64_t count, double lo, double hi,
                     double* out) {
  const uint64_t key = col_key(seed, matrix, 0);
  for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * u01(key, uint64_t(i));
}

}  // extern "C"
