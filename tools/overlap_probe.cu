// Do FP64 DMMA (mma.sync m8n8k4) and int8 tcgen05.mma run concurrently on one
// SM?  (Measured: no — both alone 2.74 / 1.40 ms, together 4.13 ms: they
// share the tensor datapath, so fusing the S_BR and linear-term launches
// cannot overlap them.)  One CTA per SM: warps 4..7 issue DMMA chains, warp 1 (one thread)
// issues tcgen05.mma.kind::i8 M128 N256 K32 from resident smem; each side is
// timed alone and together (same iteration counts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_1210_7683_b200/csrc overlap_probe.cu -o overlap_probe
#include <cstdio>
#include <cuda_runtime.h>

#include "i8_core.cuh"

using namespace gwg;
using C = I8Tile<32>;

__global__ void __launch_bounds__(256, 1) probe(int mode, int dmma_iters, int mma_iters,
                                                double* sink, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::STAGE_BYTES);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < int(C::STAGE_BYTES / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot)), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const long long t0 = clock64();
  if (warp == 1 && (mode & 2) && threadIdx.x == 32) {
    constexpr uint32_t idesc = i8_instr_desc<C::BN, C::BM>();
    const uint32_t sa = smem_u32(base), sb = sa + C::A_BYTES;
    uint32_t phase = 0;
    for (int it = 0; it < mma_iters; ++it) {
#pragma unroll 1
      for (int k = 0; k < 64; ++k)
        umma_i8(tmem + uint32_t((k & 1) * C::BN), umma_desc_sw128(sa + (k & 3) * 32),
                umma_desc_sw128(sb + (k & 3) * 32), idesc, 1u);
      umma_commit(bar);
      mbar_wait(bar, phase);
      phase ^= 1;
    }
  }
  if (warp >= 4 && (mode & 1)) {
    double acc[16][2];
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int it = 0; it < dmma_iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) dmma_ordered(acc[i], a, b);
    }
    double s = 0.0;
    for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) sink[0] = s;
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512)
                 : "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 8);
  cudaMallocManaged(&cyc, sms * sizeof(long long));
  const size_t smem = C::STAGE_BYTES + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int dmma_iters = 20000, mma_iters = 300;
  const char* names[4] = {"", "dmma alone", "i8 mma alone", "both"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 1; mode <= 3; ++mode) {
    probe<<<sms, 256, smem>>>(mode, 100, 5, sink, cyc);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    probe<<<sms, 256, smem>>>(mode, dmma_iters, mma_iters, sink, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);

    // DMMA: sms x 4 warps x 16 x iters x 512 flop; i8: sms x 64 x iters x 2*128*256*32 ops
    const double dmma_tf = double(sms) * 4 * 16 * dmma_iters * 512 / (ms * 1e-3) / 1e12;
    const double i8_tops = double(sms) * 64 * mma_iters * 2.0 * 128 * 256 * 32 / (ms * 1e-3) / 1e12;
    printf("{\"run\": \"%s\", \"ms\": %.3f, \"dmma_tflops\": %.1f, \"i8_tops\": %.0f, \"err\": \"%s\"}\n",
           names[mode], ms, (mode & 1) ? dmma_tf : 0.0, (mode & 2) ? i8_tops : 0.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
