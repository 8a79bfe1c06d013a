// int8 tensor-core peak on this B200 (sm_100a): tcgen05.mma kind::i8,
// M128 x N256 x K32 per instruction, operands resident in shared memory (no
// TMA in the loop), accumulators in TMEM — the ceiling for rotate_i8_kernel and
// linear_solve_kernel.  One CTA per SM, one issuing thread, commits every 64
// MMAs to bound the async queue.  Issue modes: one thread in a lane-0 branch,
// or the whole warp with one lane elected per instruction (the faster form).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_1210_7683_b200/csrc i8_peak.cu -o i8_peak
#include <cstdio>
#include <cuda_runtime.h>

#include "i8_core.cuh"

using namespace gwg;
using C = I8Tile<32>;

// MODE 0: consecutive MMAs alternate two accumulators, one commit per 64;
// 1: one accumulator (a GEMM's K loop); MODE >= 2: 1 plus a commit every MODE
// MMAs (4 = one operand stage of the int8 kernels) to a barrier nobody waits on
template <int BN, int MODE = 0>
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters, int* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::STAGE_BYTES);
  uint64_t* bar2 = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < int(C::STAGE_BYTES / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar2, 1);
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
  if (MODE >= 100 && warp == 1) {
    // the whole warp runs the loop (warp-uniform descriptors in uniform
    // registers); one elected lane issues each MMA / commit
    constexpr uint32_t idesc = i8_instr_desc<BN, C::BM>();
    const uint32_t sa = smem_u32(base), sb = sa + C::A_BYTES;
    const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sb);
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int k = 0; k < 64; ++k) {
        asm volatile(
            "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n}\n" ::"r"(tmem),
            "l"(da + uint64_t((k & 3) * 2)), "l"(db + uint64_t((k & 3) * 2)), "r"(idesc)
            : "memory");
        if (MODE > 100 && (k % (MODE - 100)) == MODE - 101 && k != 63)
          asm volatile(
              "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
              ::"r"(smem_u32(bar2)) : "memory");
      }
      asm volatile(
          "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
          ::"r"(smem_u32(bar)) : "memory");
      mbar_wait(bar, phase);
      phase ^= 1;
    }
  } else if (MODE < 100 && threadIdx.x == 32) {
    constexpr uint32_t idesc = i8_instr_desc<BN, C::BM>();
    const uint32_t sa = smem_u32(base), sb = sa + C::A_BYTES;  // B: up to 256 rows
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int k = 0; k < 64; ++k) {
        umma_i8(tmem + uint32_t(MODE == 0 ? (k & 1) * BN : 0), umma_desc_sw128(sa + (k & 3) * 32),
                umma_desc_sw128(sb + (k & 3) * 32), idesc, 1u);
        if (MODE >= 2 && (k % MODE) == MODE - 1 && k != 63) umma_commit(bar2);
      }
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
  const size_t smem = C::A_BYTES + 256 * C::BK + 2048;
  cudaFuncSetAttribute(i8_peak_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(i8_peak_kernel<224>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(i8_peak_kernel<224, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(i8_peak_kernel<224, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(i8_peak_kernel<224, 100>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(i8_peak_kernel<256, 100>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(i8_peak_kernel<224, 104>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("# NVIDIA B200 SMs=%d clock=%d kHz; tcgen05.mma.kind::i8 M%d N{256,224} K%d\n", sms, clk,
         C::BM, C::UK);
  for (int v : {0, 1, 2, 3, 4, 5, 6}) {
    const int bn = v == 0 || v == 6 ? 256 : 224;
    auto kern = v == 0 ? i8_peak_kernel<256> : v == 1 ? i8_peak_kernel<224>
                : v == 2 ? i8_peak_kernel<224, 1> : v == 3 ? i8_peak_kernel<224, 4>
                : v == 4 ? i8_peak_kernel<224, 100> : v == 5 ? i8_peak_kernel<224, 104>
                : i8_peak_kernel<256, 100>;
    const char* modes[7] = {"two accumulators (one thread)", "two accumulators (one thread)",
                            "one accumulator (one thread)",
                            "one accumulator, commit per 4 (one thread)",
                            "one accumulator (warp, elect.sync)",
                            "one accumulator, commit per 4 (warp, elect.sync)",
                            "one accumulator (warp, elect.sync)"};
    const char* mode = modes[v];
    for (int iters : {2000, 8000}) {
      kern<<<sms, 128, smem>>>(20, sink);  // warm-up
      cudaEventRecord(e0);
      kern<<<sms, 128, smem>>>(iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * C::BM * bn * C::UK * 64.0 * iters * sms;
      printf("{\"kernel\": \"tcgen05_i8_m128n%dk32\", \"mode\": \"%s\", \"ctas\": %d, "
             "\"mmas_per_cta\": %d, \"ms\": %.3f, \"tops\": %.1f, \"err\": \"%s\"}\n",
             bn, mode, sms, 64 * iters, ms, ops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
