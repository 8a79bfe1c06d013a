// Probe: HBM write bandwidth of the result-store pattern.  3.2 GB (one c1
// step of b) written as contiguous pieces of `piece` bytes; piece q of a
// "row" r lands at r * stride + q * piece, rows written round-robin, the way
// linear_solve_kernel's tiles write 32-SNP x p segments of many trait rows of
// the stream layout (j*m + i)*p concurrently.  Each warp writes one piece per
// step with 256-bit stores, L2 evict_first or evict_normal.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/write_bw tools/write_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__global__ void writer(double* out, int64_t pieces, int64_t piece_doubles, int64_t rows,
                       int64_t stride_doubles, int first) {
  const uint64_t pol = first ? pol_first() : pol_normal();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = warp; q < pieces; q += warps) {
    const int64_t r = q % rows, c = q / rows;
    double* base = out + r * stride_doubles + c * piece_doubles;
    for (int64_t o = lane * 4; o < piece_doubles; o += 128) {
      const double v = double(q + o);
      asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %1, %1, %1}, %2;" ::"l"(base + o),
                   "d"(v), "l"(pol)
                   : "memory");
    }
  }
}

int main() {
  const int64_t total = 3200000000ll;  // bytes
  double* out = nullptr;
  if (cudaMalloc(&out, size_t(total) + (64 << 20)) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t pieces_list[] = {256, 1024, 4096, 16384, 65536, 1 << 20};
  for (int first = 1; first >= 0; --first)
    for (int64_t piece : pieces_list)
      for (int64_t rows : {int64_t(1000), int64_t(1)}) {
        // rows: 1000 trait rows of total/1000 bytes each (the stream layout at
        // c1: 3.2 MB per trait row), or one sequential row
        const int64_t row_bytes = total / rows;
        if (piece > row_bytes) continue;
        const int64_t pieces = total / piece;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(a);
          writer<<<sms * 4, 256>>>(out, pieces, piece / 8, rows, row_bytes / 8, first);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          if (rep > 0 && ms < best) best = ms;
        }
        printf("{\"policy\": \"%s\", \"piece_bytes\": %lld, \"rows\": %lld, \"ms\": %.3f, \"tbs\": %.2f}\n",
               first ? "evict_first" : "evict_normal", (long long)piece, (long long)rows, best,
               total / (best * 1e-3) / 1e12);
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
