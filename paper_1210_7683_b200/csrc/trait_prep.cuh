// trait_prep.cuh — per-trait context kernel (K2).
//
// Replaces build_trait_weights + build_trait_context + build_trait_contexts
// (proj/src/gls.cpp:48-103, proj/src/grid.cpp:146-175).  One CTA per trait j:
//   d_k  = sigma2_j (h2_j lambda_k + (1 - h2_j))       (gls.cpp:55-57)
//   relative floor: every d_k > 1e-13 max d, else the trait fails
//                   (NotPositiveDefiniteError(-1, j), gls.cpp:59-75)
//   D_k  = 1 / d_k  (= k_k^2 of the reference)
//   trait-operand panel columns: D.X_L'_c (c < p-1), D.Y'_j, D
//   S_TL = X_L'^T diag(D) X_L' (lower), b_T = X_L'^T diag(D) Y'_j
//   chol(S_TL) in Eigen's unblocked LLT order, z_T = L^-1 b_T
// The panel is written in the exact shared-memory stage order the grid kernel
// consumes ([tile][kc][c][g][jj][kk]), so the grid kernel moves it with one
// bulk copy per stage.
#pragma once

#include "grid_kernel.cuh"

namespace gwg {

struct PrepArgs {
  int64_t n;
  int64_t np;
  int32_t t;
  const double* lambda;
  const double* y;      // rotated traits, column j at y + j * ldy
  int64_t ldy;
  const double* xl;     // rotated covariates, column c at xl + c * ldxl
  int64_t ldxl;
  const double* h2;
  const double* sigma2;
  double* bops;
  double* ctx;
  unsigned long long* trait_err;  // min j whose weights fail the floor
  int32_t panels = 1;             // write the FP64 grid's operand panels (bops)
};

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red /* [32*NV] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = v[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    v[q] = x;
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[warp * NV + q] = v[q];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = lane < nwarps ? red[lane * NV + q] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      v[q] = x;
    }
  }
  __syncthreads();
}

template <int P, int BT>
__global__ void __launch_bounds__(256) trait_prep_kernel(const PrepArgs a) {
  constexpr int P1 = P - 1;
  constexpr int NC = P + 1;
  constexpr int NQ = P1 * (P1 + 1) / 2 + P1;  // S_TL lower + b_T
  constexpr int CH = 8;                        // sums reduced per pass
  using L = CtxLayout<P>;
  __shared__ double red[32 * CH];
  __shared__ double sums[NQ > 0 ? NQ : 1];
  __shared__ double dmax_s;
  __shared__ int bad_s;

  const int j = blockIdx.x;
  const double h2 = a.h2[j], s2 = a.sigma2[j];
  const double omh = 1.0 - h2;
  const double* y = a.y + size_t(j) * a.ldy;

  // --- weights and the relative positivity floor ------------------------------
  double dmax = -INFINITY;
  for (int64_t k = threadIdx.x; k < a.n; k += blockDim.x) dmax = fmax(dmax, s2 * (h2 * a.lambda[k] + omh));
  {
    for (int off = 16; off > 0; off >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
    if (threadIdx.x == 0) bad_s = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = red[0];
      for (int w = 1; w < int(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
      dmax_s = m;
    }
    __syncthreads();
  }
  const double floor_ = 1e-13 * dmax_s;

  // --- operand panel + context sums -------------------------------------------
  const int tt = j / BT, g = (j % BT) >> 3, jj = j & 7;
  double* panel = a.bops + size_t(tt) * size_t(a.np) * NC * BT + g * 64 + jj * 8;
  for (int64_t k = threadIdx.x; k < a.np; k += blockDim.x) {
    double dinv = 0.0;
    if (k < a.n) {
      const double d = s2 * (h2 * a.lambda[k] + omh);
      if (!(d > floor_)) bad_s = 1;
      dinv = 1.0 / d;
    }
    if (!a.panels) continue;
    double* dst = panel + (k >> 3) * (NC * BT * 8) + (k & 7);
#pragma unroll
    for (int c = 0; c < P1; ++c) dst[c * BT * 8] = k < a.n ? dinv * a.xl[k + c * a.ldxl] : 0.0;
    dst[P1 * BT * 8] = k < a.n ? dinv * y[k] : 0.0;
    dst[P * BT * 8] = dinv;
  }

  for (int q0 = 0; q0 < NQ; q0 += CH) {
    double v[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) v[q] = 0.0;
    for (int64_t k = threadIdx.x; k < a.n; k += blockDim.x) {
      const double dinv = 1.0 / (s2 * (h2 * a.lambda[k] + omh));
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int qq = q0 + q;
        if (qq >= NQ) break;
        if (qq < P1 * (P1 + 1) / 2) {
          int ra = 0;
          while ((ra + 1) * (ra + 2) / 2 <= qq) ++ra;
          const int cb = qq - ra * (ra + 1) / 2;
          v[q] += (dinv * a.xl[k + ra * a.ldxl]) * a.xl[k + cb * a.ldxl];
        } else {
          const int ra = qq - P1 * (P1 + 1) / 2;
          v[q] += (dinv * a.xl[k + ra * a.ldxl]) * y[k];
        }
      }
    }
    block_sum<CH>(v, red);
    if (threadIdx.x == 0)
#pragma unroll
      for (int q = 0; q < CH; ++q)
        if (q0 + q < NQ) sums[q0 + q] = v[q];
    __syncthreads();
  }

  __syncthreads();
  if (threadIdx.x == 0) {
    if (bad_s) atomicMin(a.trait_err, (unsigned long long)j);
    double* cx = a.ctx + size_t(j) * L::STRIDE;
    constexpr int LD = P1 > 0 ? P1 : 1;
    double l[LD * LD];
    double z[LD];
    for (int r = 0; r < P1; ++r)
      for (int c = 0; c <= r; ++c) l[r * LD + c] = sums[r * (r + 1) / 2 + c];
    for (int r = 0; r < P1; ++r) z[r] = sums[P1 * (P1 + 1) / 2 + r];
    bool ok = true;
    // Eigen llt_inplace<.., Lower>::unblocked
    for (int k = 0; k < P1 && ok; ++k) {
      double x = l[k * LD + k];
      double sq = 0.0;
      for (int c = 0; c < k; ++c) sq += l[k * LD + c] * l[k * LD + c];
      x -= sq;
      if (x <= 0.0) { ok = false; break; }
      x = sqrt(x);
      l[k * LD + k] = x;
      for (int r = k + 1; r < P1; ++r) {
        double acc = 0.0;
        for (int c = 0; c < k; ++c) acc += l[r * LD + c] * l[k * LD + c];
        l[r * LD + k] = (l[r * LD + k] - acc) / x;
      }
    }
    if (ok) {
      for (int k = 0; k < P1; ++k) {  // forward substitution, column oriented
        z[k] /= l[k * LD + k];
        for (int r = k + 1; r < P1; ++r) z[r] -= z[k] * l[r * LD + k];
      }
      for (int r = 0; r < P1; ++r) {
        cx[L::INVD + r] = 1.0 / l[r * LD + r];
        cx[L::Z + r] = z[r];
        for (int c = 0; c < r; ++c) cx[L::OFF + L::off_idx(r, c)] = l[r * LD + c];
      }
      // L^-1, column by column (forward substitution on the unit vectors)
      for (int c = 0; c < P1; ++c) {
        for (int r = c; r < P1; ++r) {
          double v = r == c ? 1.0 : 0.0;
          for (int q = c; q < r; ++q) v -= l[r * LD + q] * cx[L::LINV + L::linv_idx(q, c)];
          cx[L::LINV + L::linv_idx(r, c)] = v / l[r * LD + r];
        }
      }
      // c_T = L^-T z = S_TL^-1 b_T (back substitution) for the folded solve
      for (int r = P1 - 1; r >= 0; --r) {
        double v = z[r];
        for (int q = r + 1; q < P1; ++q) v -= l[q * LD + r] * cx[L::CT + q];
        cx[L::CT + r] = v / l[r * LD + r];
      }
    }
    cx[L::FLAG] = ok ? 0.0 : 1.0;
  }
}

// Relayout-free SNP path needs nothing else; this kernel only exists for the
// trait side.  Launch helper.
template <int P, int BT>
inline cudaError_t launch_trait_prep(const PrepArgs& a, cudaStream_t s) {
  prefer_max_smem(trait_prep_kernel<P, BT>);
  trait_prep_kernel<P, BT><<<a.t, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace gwg
