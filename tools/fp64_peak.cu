// FP64 peak microbenchmark for B200 (sm_100a): DMMA shapes vs DFMA.
// Measures the denominators for the GLS-grid roofline (MEASURED_PEAKS.json
// holds only bf16 and HBM).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int kChains = 8;

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-9;
  double c[kChains][4];
#pragma unroll
  for (int i = 0; i < kChains; ++i) for (int q = 0; q < 4; ++q) c[i][q] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = 1.0 + (threadIdx.x + q) * 1e-9;
#pragma unroll
  for (int q = 0; q < 4; ++q) b[q] = 1.0 - (threadIdx.x + q) * 1e-9;
  double c[kChains][4];
#pragma unroll
  for (int i = 0; i < kChains; ++i) for (int q = 0; q < 4; ++q) c[i][q] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
int run(const char* name, K kern, double flops_per_warp_iter, int blocks, int threads, int iters,
        double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out, iters);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double warps = double(blocks) * threads / 32;
  const double flops = warps * iters * flops_per_warp_iter;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", name,
         blocks, threads, best, flops / best / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("# %s SMs=%d clock=%d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int sms = prop.multiProcessorCount;
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      run("dmma_m8n8k4", dmma_m8n8k4, kChains * 512.0, sms * bps, warps * 32, iters, out);
      run("dmma_m16n8k4", dmma_m16n8k4, kChains * 1024.0, sms * bps, warps * 32, iters / 2, out);
      run("dmma_m16n8k16", dmma_m16n8k16, kChains * 4096.0, sms * bps, warps * 32, iters / 8, out);
      run("dfma", dfma_loop, kChains * 64.0, sms * bps, warps * 32, iters * 4, out);
    }
  }
  return 0;
}
