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
  int32_t y_only = 0;   // factorised W build: only the D.Y'_j columns, no D panels
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
    if (!a.y_only) {
      panel[(k >> 3) * (int64_t(a.bt) * 8) + (k & 7)] = dinv;
      for (int c = 0; c + 1 < a.p; ++c) v[c * a.np + k] = in ? dinv * a.xl[k + c * a.ldxl] : 0.0;
    }
    v[(a.p - 1) * a.np + k] = in ? dinv * y[k] : 0.0;
  }
}

// Fold L_j^-1 into the trait's W columns (the genotype grid's linear terms),
// so linear_solve_kernel's MMA yields the solve's intermediates directly:
//   W'_c = sum_{d<=c} (L^-1)_{c,d} W_d   (c < p-1:  x^T W'_c = (L^-1 s_bl)_c)
//   W'_y = W_y - sum_c z_c W'_c           (x^T W'_y = b_B - l.z_T)
// in place, one CTA per trait, a thread per row (descending c keeps the
// W_d it reads intact).  A trait whose chol(S_TL) failed is left as it is
// (its cells fail through the context flag).
struct FoldArgs {
  double* w;          // W columns (ld np) at (j/kt)*rb + (j%kt)*p8 + c
  int64_t n, np;
  int32_t t, p, kt, p8, rb;
  const double* ctx;  // CtxLayout<p> per trait
  int32_t stride, z, flag, linv;
};
__global__ void __launch_bounds__(256) fold_w_kernel(const FoldArgs a) {
  const int j = blockIdx.x;
  const double* cx = a.ctx + size_t(j) * a.stride;
  if (cx[a.flag] != 0.0) return;
  const int p1 = a.p - 1;
  double* w = a.w + (size_t(j / a.kt) * a.rb + size_t(j % a.kt) * a.p8) * a.np;
  for (int64_t k = threadIdx.x; k < a.n; k += blockDim.x) {
    for (int c = p1 - 1; c >= 0; --c) {
      double v = 0.0;
      for (int d = 0; d <= c; ++d) v = fma(cx[a.linv + c * (c + 1) / 2 + d], w[d * a.np + k], v);
      w[c * a.np + k] = v;
    }
    double y = w[p1 * a.np + k];
    for (int c = 0; c < p1; ++c) y = fma(-cx[a.z + c], w[c * a.np + k], y);
    w[p1 * a.np + k] = y;
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


// ---- low-rank S_BR (expsum.cpp): D = E F with positive factors ------------------

// Range of the factorisation, one CTA (256 threads: it fits beside the code
// conversion on a busy SM):
//   out[0] = min lambda, out[1] = max lambda,
//   out[2] / out[3] = min / max of gamma_j = (1 - h_j) / h_j over traits with h_j != 0,
//   out[4] = number of such traits, out[5] = 1 if some trait's scale
//   1 / (sigma2 h) (or 1 / sigma2 at h = 0) or gamma is not finite.
__global__ void __launch_bounds__(1024) expsum_range_kernel(const double* __restrict__ lambda,
                                                            int64_t n, const double* __restrict__ h2,
                                                            const double* __restrict__ sigma2,
                                                            int32_t t, double* __restrict__ out) {
  __shared__ double red[5][32];
  double v[5] = {INFINITY, -INFINITY, INFINITY, -INFINITY, 0.0};
  bool bad = false;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    v[0] = fmin(v[0], lambda[k]);
    v[1] = fmax(v[1], lambda[k]);
    bad |= !isfinite(lambda[k]);
  }
  for (int j = threadIdx.x; j < t; j += blockDim.x) {
    const double h = h2[j], s2 = sigma2[j];
    if (h != 0.0) {
      const double g = (1.0 - h) / h;
      v[2] = fmin(v[2], g);
      v[3] = fmax(v[3], g);
      v[4] += 1.0;
      bad |= !isfinite(g) || !isfinite(1.0 / (s2 * h));
    } else {
      bad |= !isfinite(1.0 / s2);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int off = 16; off > 0; off >>= 1) {
    v[0] = fmin(v[0], __shfl_xor_sync(0xffffffffu, v[0], off));
    v[1] = fmax(v[1], __shfl_xor_sync(0xffffffffu, v[1], off));
    v[2] = fmin(v[2], __shfl_xor_sync(0xffffffffu, v[2], off));
    v[3] = fmax(v[3], __shfl_xor_sync(0xffffffffu, v[3], off));
    v[4] += __shfl_xor_sync(0xffffffffu, v[4], off);
  }
  const bool any_bad = __syncthreads_or(bad);
  if (lane == 0)
    for (int q = 0; q < 5; ++q) red[q][warp] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
      v[0] = fmin(v[0], red[0][w]);
      v[1] = fmax(v[1], red[1][w]);
      v[2] = fmin(v[2], red[2][w]);
      v[3] = fmax(v[3], red[3][w]);
      v[4] += red[4][w];
    }
    for (int q = 0; q < 5; ++q) out[q] = v[q];
    out[5] = any_bad ? 1.0 : 0.0;
  }
}

struct ExpSumArgs {
  int64_t n;
  int64_t np;
  int32_t t;
  int32_t r;            // terms (multiple of bt)
  int32_t bt;           // gls_sbr_kernel panel width
  const double* lambda;
  const double* h2;
  const double* sigma2;
  const double* s;      // nodes s_r (s_0 = 0)
  const double* w;      // weights w_r
  double lam0;          // min lambda
  double* epanel;       // E[k][r] = exp(-s_r (lambda_k - lam0)) as D panels over r
  double* fpanel;       // F[r][j] = w_r exp(-s_r (lam0 + gamma_j)) / (sigma2_j h_j)
  // expsum_e_kernel with xmul: columns c * r + q of panel_out (ld ldx per c)
  // hold x_c[k] E[k][q] for c < ncx (the W build's diag(X_L'_c) E)
  const double* xmul = nullptr;
  int64_t ldx = 0;
  int32_t ncx = 0;
  double* panel_out = nullptr;
};

// D-panel index ([tile][k/8][column octet][column%8][k%8]) of (k, column c).
__device__ __forceinline__ size_t panel_index(int64_t k, int64_t c, int32_t bt, int64_t kext) {
  return size_t(c / bt) * size_t(kext) * bt + size_t(k >> 3) * (size_t(bt) * 8) +
         size_t((c % bt) >> 3) * 64 + size_t(c & 7) * 8 + size_t(k & 7);
}

// exp(-s x) with the rounding of the product s x compensated: exp is
// conditioned by s x (up to ~39 on the terms that matter), so an
// uncompensated product would cost ~39 ulps per term; the errors of x itself
// are common to all terms of a sum and cost only their own size.
__device__ __forceinline__ double exp_neg_prod(double s, double x) {
  const double hi = s * x;
  const double lo = fma(s, x, -hi);  // s x = hi + lo exactly
  return exp(-hi) * (1.0 - lo);
}

// One CTA per term r: column r of E, the K operand of GEMM 1 (K = eigen-rows).
// With xmul: one CTA per (c, r), column c * r + q of panel_out = x_c . E_q.
__global__ void __launch_bounds__(256) expsum_e_kernel(const ExpSumArgs a) {
  const int col = blockIdx.x;
  const int q = a.xmul ? col % a.r : col;
  const int c = a.xmul ? col / a.r : 0;
  const double s = a.s[q];
  double* out = a.xmul ? a.panel_out : a.epanel;
  const double* x = a.xmul ? a.xmul + int64_t(c) * a.ldx : nullptr;
  for (int64_t k = threadIdx.x; k < a.np; k += blockDim.x) {
    double v = k < a.n ? exp_neg_prod(s, a.lambda[k] - a.lam0) : 0.0;
    if (x) v = k < a.n ? v * x[k] : 0.0;
    out[panel_index(k, col, a.bt, a.np)] = v;
  }
}

// One CTA per trait j: column j of F, the K operand of GEMM 2 (K = terms).
// h_j = 0 (D constant 1 / sigma2) uses only the constant term (s_0 = 0).
__global__ void __launch_bounds__(128) expsum_f_kernel(const ExpSumArgs a) {
  const int j = blockIdx.x;
  const double h = a.h2[j], s2 = a.sigma2[j];
  const double coef = h != 0.0 ? 1.0 / (s2 * h) : 1.0 / s2;
  const double beta = h != 0.0 ? a.lam0 + (1.0 - h) / h : 0.0;
  for (int r = threadIdx.x; r < a.r; r += blockDim.x) {
    double f;
    if (h != 0.0)
      f = (a.w[r] * coef) * exp_neg_prod(a.s[r], beta);
    else
      f = r == 0 ? coef : 0.0;
    a.fpanel[panel_index(r, j, a.bt, a.r)] = f;
  }
}

}  // namespace gwg
