// verify.cu — device Cholesky-route verifier.
//
// The reference checks grids with an independent route that never touches the
// eigendecomposition: CholeskyOracle (proj/src/gls.cpp:188-244) forms
// M = sigma2 (h2 Phi + (1 - h2) I), factors it (LLT), solves u = L^-1 X,
// z = L^-1 y and the p x p normal equations; gwgrid.verify_grid
// (proj/python/bindings.cpp:192-222) and `gwgrid verify`
// (tools/gwgrid_main.cpp:315-400) report the max norm-wise relative error
// |b - ref| / |ref| over cells.  Here, per trait j:
//   M_j built by a kernel, potrf (cuSOLVER), W = L^-1 [X_L | y_j | X_R] (cuBLAS
//   trsm), G = W_R^T [W_L | w_y] (cuBLAS gemm), then one thread per SNP
//   assembles and LLT-solves its p x p system and compares with b.
// Library factorizations are fine here: this is the checker, not the hot path.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/gwgrid_cuda.h"

namespace {

constexpr int kMaxP = 32;

int fail(gwg_status* st, int code, int64_t snp, int64_t trait, const char* fmt, ...) {
  if (st) {
    st->code = code;
    st->snp_index = snp;
    st->trait_index = trait;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

__global__ void build_m_kernel(const double* __restrict__ phi, int64_t n, double a, double b,
                               double* __restrict__ m) {
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    m[idx] = phi[idx] * a + (i == j ? b : 0.0);
  }
}

// One thread per SNP column i of the slab: S = [[S_LL, g_i(0:p-1)], [.., |w_i|^2]],
// rhs = [r_L ; g_i(p-1)], LLT solve, norm-wise error against b(i, j).
__global__ void cells_kernel(int64_t n, int p, int64_t m, const double* __restrict__ w,
                             int64_t ldw, const double* __restrict__ g, int64_t ldg,
                             const double* __restrict__ sll, const double* __restrict__ rl,
                             const double* __restrict__ b, int64_t b_si, double* err_out,
                             double* cell_err, int64_t cell_si, int* npd_out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const int pm1 = p - 1;
  const double* wi = w + (pm1 + 1 + i) * ldw;  // column of L^-1 x_i
  double nrm = 0.0;
  for (int64_t k = 0; k < n; ++k) nrm = fma(wi[k], wi[k], nrm);
  double s[kMaxP * kMaxP], r[kMaxP];
  for (int a = 0; a < pm1; ++a) {
    for (int c = 0; c < pm1; ++c) s[a * p + c] = sll[a + c * pm1];
    r[a] = rl[a];
    s[pm1 * p + a] = s[a * p + pm1] = g[i + a * ldg];
  }
  s[pm1 * p + pm1] = nrm;
  r[pm1] = g[i + pm1 * ldg];
  // LLT (row-major lower in s)
  for (int k = 0; k < p; ++k) {
    double x = s[k * p + k];
    for (int c = 0; c < k; ++c) x -= s[k * p + c] * s[k * p + c];
    if (!(x > 0.0)) {
      atomicMax(npd_out, 1);
      return;
    }
    x = sqrt(x);
    s[k * p + k] = x;
    for (int q = k + 1; q < p; ++q) {
      double v = s[q * p + k];
      for (int c = 0; c < k; ++c) v -= s[q * p + c] * s[k * p + c];
      s[q * p + k] = v / x;
    }
  }
  for (int k = 0; k < p; ++k) {
    double v = r[k];
    for (int c = 0; c < k; ++c) v -= s[k * p + c] * r[c];
    r[k] = v / s[k * p + k];
  }
  for (int k = p - 1; k >= 0; --k) {
    double v = r[k];
    for (int c = k + 1; c < p; ++c) v -= s[c * p + k] * r[c];
    r[k] = v / s[k * p + k];
  }
  double d2 = 0.0, r2 = 0.0;
  const double* bi = b + i * b_si;
  for (int c = 0; c < p; ++c) {
    const double d = bi[c] - r[c];
    d2 += d * d;
    r2 += r[c] * r[c];
  }
  const double rel = r2 > 0.0 ? sqrt(d2 / r2) : sqrt(d2);
  if (cell_err) cell_err[i * cell_si] = rel;
  atomicMax(reinterpret_cast<unsigned long long*>(err_out),
            static_cast<unsigned long long>(__double_as_longlong(rel)));
}

}  // namespace

extern "C" int32_t gwg_verify_grid(int32_t device, int64_t n, int64_t p, int64_t m, int64_t t,
                                   const double* kinship, const double* xl, const double* snps,
                                   const double* traits, const double* h2, const double* sigma2,
                                   const double* b, double* cell_err, double* max_rel_err,
                                   gwg_status* st) {
  if (st) {
    st->code = GWG_OK;
    st->snp_index = st->trait_index = -1;
    st->msg[0] = 0;
  }
  if (n < 1 || p < 1 || p > n || p > kMaxP || m < 1 || t < 1 || !kinship || !snps || !traits ||
      !h2 || !sigma2 || !b || !max_rel_err || (p > 1 && !xl))
    return fail(st, GWG_DIMENSION, -1, -1, "bad verify_grid arguments");
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return fail(st, GWG_CUDA, -1, -1, "CUDA device %d not available", device);
  }
  const int64_t pm1 = p - 1, wc = pm1 + 1 + m;
  std::vector<void*> bufs;
  auto dalloc = [&](size_t bytes) -> double* {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(bytes, 8)) != cudaSuccess) return nullptr;
    bufs.push_back(q);
    return static_cast<double*>(q);
  };
  double* d_phi = dalloc(size_t(n) * n * 8);
  double* d_m = dalloc(size_t(n) * n * 8);
  double* d_src = dalloc(size_t(n) * wc * 8);   // [X_L | (y) | X_R] raw, y slot per trait
  double* d_w = dalloc(size_t(n) * wc * 8);
  double* d_g = dalloc(size_t(m) * p * 8);
  double* d_sl = dalloc(size_t(p) * p * 8);
  double* d_b = dalloc(size_t(m) * t * p * 8);
  double* d_y = dalloc(size_t(n) * t * 8);
  double* d_err = dalloc(8);
  double* d_cell = cell_err ? dalloc(size_t(m) * t * 8) : nullptr;
  int* d_npd = reinterpret_cast<int*>(dalloc(8));
  cusolverDnHandle_t sh = nullptr;
  cublasHandle_t bh = nullptr;
  int* d_info = reinterpret_cast<int*>(dalloc(8));
  int32_t rc = GWG_OK;
  auto cleanup = [&] {
    if (sh) cusolverDnDestroy(sh);
    if (bh) cublasDestroy(bh);
    for (void* q : bufs) cudaFree(q);
  };
  for (void* q : bufs)
    if (!q) {
      cleanup();
      return fail(st, GWG_CUDA, -1, -1, "cudaMalloc failed in verify_grid");
    }
  if (cusolverDnCreate(&sh) != CUSOLVER_STATUS_SUCCESS ||
      cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) {
    cleanup();
    return fail(st, GWG_BACKEND, -1, -1, "cuSOLVER/cuBLAS init failed");
  }
  cublasSetMathMode(bh, CUBLAS_PEDANTIC_MATH);
  cudaMemcpy(d_phi, kinship, size_t(n) * n * 8, cudaMemcpyHostToDevice);
  if (pm1) cudaMemcpy(d_src, xl, size_t(n) * pm1 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_src + (pm1 + 1) * n, snps, size_t(n) * m * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_y, traits, size_t(n) * t * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_b, b, size_t(m) * t * p * 8, cudaMemcpyHostToDevice);
  cudaMemset(d_err, 0, 8);
  cudaMemset(d_npd, 0, 4);
  int lwork = 0;
  cusolverDnDpotrf_bufferSize(sh, CUBLAS_FILL_MODE_LOWER, int(n), d_m, int(n), &lwork);
  double* d_work = dalloc(size_t(std::max(lwork, 1)) * 8);
  if (!d_work) {
    cleanup();
    return fail(st, GWG_CUDA, -1, -1, "cudaMalloc failed in verify_grid");
  }
  const double one = 1.0, zero = 0.0;
  for (int64_t j = 0; j < t && rc == GWG_OK; ++j) {
    // M_j = sigma2 (h2 Phi + (1 - h2) I)   (gls.cpp:195-196)
    build_m_kernel<<<1184, 256>>>(d_phi, n, sigma2[j] * h2[j], sigma2[j] * (1.0 - h2[j]), d_m);
    if (cusolverDnDpotrf(sh, CUBLAS_FILL_MODE_LOWER, int(n), d_m, int(n), d_work, lwork,
                         d_info) != CUSOLVER_STATUS_SUCCESS) {
      rc = fail(st, GWG_BACKEND, -1, j, "potrf failed");
      break;
    }
    int info = 0;
    cudaMemcpy(&info, d_info, 4, cudaMemcpyDeviceToHost);
    if (info != 0) {
      rc = fail(st, GWG_NOT_POSITIVE_DEFINITE, -1, j,
                "trait covariance is not positive definite (trait %lld)", (long long)j);
      break;
    }
    cudaMemcpy(d_src + pm1 * n, d_y + j * n, size_t(n) * 8, cudaMemcpyDeviceToDevice);
    cudaMemcpy(d_w, d_src, size_t(n) * wc * 8, cudaMemcpyDeviceToDevice);
    cublasDtrsm(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                int(n), int(wc), &one, d_m, int(n), d_w, int(n));
    // G = W_R^T [W_L | w_y]  (m x p);  S_LL | r_L = W_L^T [W_L | w_y]  (pm1 x p)
    cublasDgemm(bh, CUBLAS_OP_T, CUBLAS_OP_N, int(m), int(p), int(n), &one,
                d_w + (pm1 + 1) * n, int(n), d_w, int(n), &zero, d_g, int(m));
    if (pm1)
      cublasDgemm(bh, CUBLAS_OP_T, CUBLAS_OP_N, int(pm1), int(p), int(n), &one, d_w, int(n), d_w,
                  int(n), &zero, d_sl, int(pm1));
    cells_kernel<<<int((m + 127) / 128), 128>>>(n, int(p), m, d_w, n, d_g, m, d_sl,
                                                d_sl + pm1 * pm1, d_b + j * p, t * p, d_err,
                                                d_cell ? d_cell + j : nullptr, t, d_npd);
  }
  if (rc == GWG_OK) {
    cudaError_t ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) rc = fail(st, GWG_CUDA, -1, -1, "%s", cudaGetErrorString(ce));
  }
  if (rc == GWG_OK) {
    int npd = 0;
    cudaMemcpy(max_rel_err, d_err, 8, cudaMemcpyDeviceToHost);
    if (d_cell) cudaMemcpy(cell_err, d_cell, size_t(m) * t * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&npd, d_npd, 4, cudaMemcpyDeviceToHost);
    if (npd)
      rc = fail(st, GWG_NOT_POSITIVE_DEFINITE, -1, -1,
                "oracle normal equations are not positive definite");
  }
  cleanup();
  return rc;
}
