// eig.cu — device eigendecomposition of the kinship matrix.
//
// Same contract as eigendecompose_kinship (proj/src/gls.cpp:16-46):
//   symmetry gate  max|Phi - Phi^T| <= 1e-12 max|Phi|  else NonSymmetricError
//   Phi = Z diag(lambda) Z^T, lambda ascending, orthonormal Z
//   sign rule      each column's largest-magnitude entry (first on ties) > 0
// The symmetric solve itself is cuSOLVER's syevd (a library routine, like the
// reference's Eigen SelfAdjointEigenSolver); the gate and the sign rule are
// this file's kernels.  The grid itself never depends on which eigensolver
// produced Z: it consumes any orthonormal eigenbasis.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/gwgrid_cuda.h"

namespace {

int fail(gwg_status* st, int code, const char* fmt, ...) {
  if (st) {
    st->code = code;
    st->snp_index = -1;
    st->trait_index = -1;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

// Non-negative doubles order like their bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
  atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void sym_gate_kernel(const double* __restrict__ a, int64_t n, int64_t lda,
                                unsigned long long* out /* [0]=max|a|, [1]=max|a-a^T| */) {
  double amax = 0.0, asym = 0.0;
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    const double v = a[i + j * lda];
    amax = fmax(amax, fabs(v));
    if (i > j) asym = fmax(asym, fabs(v - a[j + i * lda]));
  }
  for (int off = 16; off > 0; off >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(&out[0], amax);
    atomic_max_nonneg(&out[1], asym);
  }
}

__global__ void sign_rule_kernel(double* __restrict__ z, int64_t n, int64_t ld) {
  __shared__ double best_v[32];
  __shared__ int64_t best_i[32];
  __shared__ int flip;
  double* col = z + blockIdx.x * ld;
  double bv = -1.0;
  int64_t bi = 0;
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
    const double v = fabs(col[r]);
    if (v > bv) {  // strided scan: the first index wins ties within a thread
      bv = v;
      bi = r;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    best_v[w] = bv;
    best_i[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < int(blockDim.x >> 5); ++q)
      if (best_v[q] > bv || (best_v[q] == bv && best_i[q] < bi)) {
        bv = best_v[q];
        bi = best_i[q];
      }
    flip = col[bi] < 0.0;
  }
  __syncthreads();
  if (flip)
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) col[r] = -col[r];
}

}  // namespace

// In-place device eigendecomposition of a (n x n, ld lda, device memory):
// a <- Z, w <- lambda (device).  Used by gwg_eigendecompose and the engine.
extern "C" int32_t gwg_internal_device_eig(double* a, int64_t n, int64_t lda, double* w,
                                           cudaStream_t stream, gwg_status* st) {
  unsigned long long* gate = nullptr;
  if (cudaMalloc(&gate, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return fail(st, GWG_CUDA, "cudaMalloc failed");
  cudaMemsetAsync(gate, 0, 2 * sizeof(unsigned long long), stream);
  const int blocks = int(std::min<int64_t>((n * n + 255) / 256, 148 * 8));
  sym_gate_kernel<<<blocks, 256, 0, stream>>>(a, n, lda, gate);
  unsigned long long hg[2] = {0, 0};
  cudaMemcpyAsync(hg, gate, sizeof(hg), cudaMemcpyDeviceToHost, stream);
  cudaError_t ce = cudaStreamSynchronize(stream);
  cudaFree(gate);
  if (ce != cudaSuccess) return fail(st, GWG_CUDA, "symmetry gate: %s", cudaGetErrorString(ce));
  double scale, asym;
  std::memcpy(&scale, &hg[0], 8);
  std::memcpy(&asym, &hg[1], 8);
  if (asym > 1e-12 * scale)
    return fail(st, GWG_NON_SYMMETRIC,
                "relatedness matrix is not symmetric: max|A-A'|=%g exceeds 1e-12*max|A|=%g",
                asym, 1e-12 * scale);

  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t prm = nullptr;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS)
    return fail(st, GWG_BACKEND, "cusolverDnCreate failed");
  cusolverDnSetStream(h, stream);
  cusolverDnCreateParams(&prm);
  size_t dev_bytes = 0, host_bytes = 0;
  int32_t rc = GWG_OK;
  void* dbuf = nullptr;
  int* dinfo = nullptr;
  std::vector<char> hbuf;
  if (cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                  CUDA_R_64F, a, lda, CUDA_R_64F, w, CUDA_R_64F, &dev_bytes,
                                  &host_bytes) != CUSOLVER_STATUS_SUCCESS) {
    rc = fail(st, GWG_BACKEND, "cusolverDnXsyevd_bufferSize failed");
  } else if (cudaMalloc(&dbuf, dev_bytes + sizeof(int)) != cudaSuccess) {
    rc = fail(st, GWG_CUDA, "cudaMalloc(%zu) for syevd failed", dev_bytes);
  } else {
    dinfo = reinterpret_cast<int*>(static_cast<char*>(dbuf) + dev_bytes);
    hbuf.resize(host_bytes + 1);
    if (cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F,
                         a, lda, CUDA_R_64F, w, CUDA_R_64F, dbuf, dev_bytes, hbuf.data(),
                         host_bytes, dinfo) != CUSOLVER_STATUS_SUCCESS) {
      rc = fail(st, GWG_BACKEND, "cusolverDnXsyevd failed");
    } else {
      int info = 0;
      cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, stream);
      cudaStreamSynchronize(stream);
      if (info != 0) rc = fail(st, GWG_BACKEND, "symmetric eigensolver did not converge");
    }
  }
  if (dbuf) cudaFree(dbuf);
  if (prm) cusolverDnDestroyParams(prm);
  cusolverDnDestroy(h);
  if (rc != GWG_OK) return rc;
  sign_rule_kernel<<<int(n), 256, 0, stream>>>(a, n, lda);
  ce = cudaStreamSynchronize(stream);
  if (ce != cudaSuccess) return fail(st, GWG_CUDA, "sign rule: %s", cudaGetErrorString(ce));
  return GWG_OK;
}

extern "C" int32_t gwg_eigendecompose(int32_t device, int64_t n, const double* phi,
                                      int32_t where, double* basis, double* values,
                                      int32_t out_where, gwg_status* st) {
  if (st) {
    st->code = GWG_OK;
    st->snp_index = st->trait_index = -1;
    st->msg[0] = 0;
  }
  if (n < 1 || !phi || !basis || !values)
    return fail(st, GWG_DIMENSION, "relatedness matrix must be square and non-empty");
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return fail(st, GWG_CUDA, "CUDA device %d not available", device);
  }
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
    return fail(st, GWG_CUDA, "stream creation failed");
  double *a = nullptr, *w = nullptr;
  int32_t rc = GWG_OK;
  const size_t bytes = size_t(n) * n * sizeof(double);
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&w, n * sizeof(double)) != cudaSuccess) {
    rc = fail(st, GWG_CUDA, "cudaMalloc failed for n=%lld", (long long)n);
  } else {
    cudaMemcpyAsync(a, phi, bytes,
                    where == GWG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
    rc = gwg_internal_device_eig(a, n, n, w, s, st);
    if (rc == GWG_OK) {
      const cudaMemcpyKind k =
          out_where == GWG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      cudaMemcpyAsync(basis, a, bytes, k, s);
      cudaMemcpyAsync(values, w, n * sizeof(double), k, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) rc = fail(st, GWG_CUDA, "copy-out failed");
    }
  }
  if (a) cudaFree(a);
  if (w) cudaFree(w);
  cudaStreamDestroy(s);
  return rc;
}
