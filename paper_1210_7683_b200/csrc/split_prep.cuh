// split_prep.cuh — trait-side kernels of the split grid (grid_split.cuh):
// the V columns whose rotation gives W = Z V, the D panels of
// gls_sbr_kernel, and the Z^T copy the rotation kernel needs for W.
// Included by engine.cu only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gwg {

struct SplitPrepArgs {
  int64_t n;
  int64_t np;
  int32_t t;
  int32_t p;
  int32_t bt;           // traits per D-panel tile
  int32_t kt;           // traits per linear-solve tile (W layout, linear_solve.cuh)
  int32_t p8;           // padded columns per trait
  int32_t rb;           // W rows per linear-solve tile
  const double* lambda;
  const double* y;      // rotated traits, ld ldy
  int64_t ldy;
  const double* xl;     // rotated covariates, ld ldxl
  int64_t ldxl;
  const double* h2;
  const double* sigma2;
  double* dpanel;       // D panels for gls_sbr_kernel
  double* v;            // columns D.X_L'_c, D.Y'_j (ld np) at (j/kt)*rb + (j%kt)*p8 + c;
                        // padding columns are zeroed by the caller
};

// One CTA per trait: D_j = 1 / (sigma2 (h2 lambda + 1 - h2)) exactly as
// trait_prep_kernel computes it (same expression, so the same doubles).
__global__ void __launch_bounds__(256) split_prep_kernel(const SplitPrepArgs a) {
  const int j = blockIdx.x;
  const double h2 = a.h2[j], s2 = a.sigma2[j];
  const double omh = 1.0 - h2;
  const double* y = a.y + size_t(j) * a.ldy;
  const int tt = j / a.bt, g = (j % a.bt) >> 3, jj = j & 7;
  double* panel = a.dpanel + size_t(tt) * size_t(a.np) * a.bt + g * 64 + jj * 8;
  double* v = a.v + (size_t(j / a.kt) * a.rb + size_t(j % a.kt) * a.p8) * a.np;
  for (int64_t k = threadIdx.x; k < a.np; k += blockDim.x) {
    const bool in = k < a.n;
    const double dinv = in ? 1.0 / (s2 * (h2 * a.lambda[k] + omh)) : 0.0;
    panel[(k >> 3) * (int64_t(a.bt) * 8) + (k & 7)] = dinv;
    for (int c = 0; c + 1 < a.p; ++c) v[c * a.np + k] = in ? dinv * a.xl[k + c * a.ldxl] : 0.0;
    v[(a.p - 1) * a.np + k] = in ? dinv * y[k] : 0.0;
  }
}

// Z^T into a separate buffer (both ld np) so the DMMA rotation kernel, which
// computes Basis^T src, can form W = Z V.
__global__ void transpose_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                 int64_t n, int64_t ld) {
  __shared__ double tile[32][33];
  const int64_t bx = int64_t(blockIdx.x) * 32, by = int64_t(blockIdx.y) * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t row = bx + threadIdx.x, col = by + r;
    tile[r][threadIdx.x] = (row < n && col < n) ? src[col * ld + row] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t row = by + threadIdx.x, col = bx + r;
    if (row < n && col < n) dst[col * ld + row] = tile[threadIdx.x][r];
  }
}

}  // namespace gwg
