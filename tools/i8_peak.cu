// int8 tensor-core peak on this B200 (sm_100a): tcgen05.mma kind::i8,
// M128 x N256 x K32 per instruction, operands resident in shared memory (no
// TMA in the loop), accumulators in TMEM — the ceiling for rotate_i8_kernel and
// linear_solve_kernel.  One CTA per SM, one issuing thread, commits every 64
// MMAs to bound the async queue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_1210_7683_b200/csrc i8_peak.cu -o i8_peak
#include <cstdio>
#include <cuda_runtime.h>

#include "i8_core.cuh"

using namespace gwg;
using C = I8Tile<32>;

__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters, int* sink) {
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
                     smem_u32(slot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = i8_instr_desc<C::BN, C::BM>();
    const uint32_t sa = smem_u32(base), sb = sa + C::A_BYTES;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int k = 0; k < 64; ++k)
        umma_i8(tmem + uint32_t((k & 1) * C::BN), umma_desc_sw128(sa + (k & 3) * 32),
                umma_desc_sw128(sb + (k & 3) * 32), idesc, 1u);
      umma_commit(bar);
      mbar_wait(bar, phase);
      phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512)
                 : "memory");
  }
  if (threadIdx.x == 0) *sink = int(tmem);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int* sink;
  cudaMalloc(&sink, sizeof(int));
  const size_t smem = C::STAGE_BYTES + 2048;
  cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("# NVIDIA B200 SMs=%d clock=%d kHz; tcgen05.mma.kind::i8 M%d N%d K%d\n", sms, clk,
         C::BM, C::BN, C::UK);
  for (int iters : {200, 2000, 8000}) {
    i8_peak_kernel<<<sms, 128, smem>>>(20, sink);  // warm-up
    cudaEventRecord(e0);
    i8_peak_kernel<<<sms, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * C::BM * C::BN * C::UK * 64.0 * iters * sms;
    printf("{\"kernel\": \"tcgen05_i8_m128n256k32\", \"ctas\": %d, \"mmas_per_cta\": %d, "
           "\"ms\": %.3f, \"tops\": %.1f, \"err\": \"%s\"}\n",
           sms, 64 * iters, ms, ops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
