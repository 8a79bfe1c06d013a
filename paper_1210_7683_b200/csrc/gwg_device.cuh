// gwg_device.cuh — sm_100a device primitives used by the GLS-grid kernels:
// mbarriers, TMA (cp.async.bulk.tensor) and bulk copies, FP64 DMMA.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gwg {

// Small kernels that share SMs with 200 KB-smem CTAs (the code conversion
// under the trait-side chain, the chain's own launches): optionally prefer
// the maximum shared-memory carveout, so an SM running them need not drain
// to re-partition L1/shared memory before such a CTA joins it.  Measured
// neutral to slightly slower at c1 on its own (4.26-4.28 vs 4.25-4.27 ms):
// off.
#ifndef GWG_SMEM_CARVEOUT
#define GWG_SMEM_CARVEOUT 0
#endif
template <class Kern>
inline void prefer_max_smem(Kern* kern) {
  if (GWG_SMEM_CARVEOUT) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                         cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
    (void)cudaGetLastError();
  }
}


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// Make mbarrier inits visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Slab-path gate (GWG_SNP_AUTO): *word = ~0 when every SNP value of the slab
// is an integer genotype code (snp_to_i8_kernel), 0 otherwise.  A kernel of
// one path returns at once when the slab belongs to the other (want_codes =
// 1: genotype path, 0: FP64 path); word = null means ungated.  Uniform per
// CTA, checked before any barrier or TMEM setup.
__device__ __forceinline__ bool gate_closed(const unsigned long long* word, int32_t want_codes) {
  if (word == nullptr) return false;
  const bool codes = *reinterpret_cast<const volatile unsigned long long*>(word) == ~0ull;
  return codes != (want_codes != 0);
}

// 2-D TMA tile load into shared memory, completing on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completing on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Result store with an L2 evict_first hint: on the B200 plain stores of
// results that are not re-read made L2 fetch the written lines from HBM first
// (measured: ~0.5-1 GB of extra DRAM reads per launch at config 1).
__device__ __forceinline__ void st_evict_first(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
               : "memory");
}

// Four consecutive doubles in one 256-bit store (STG.E.ENL2.256; 32-byte
// aligned address) with an L2 cache policy.
__device__ __forceinline__ void st4_policy(double* p, double a, double b, double c, double d,
                                           uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(a),
               "d"(b), "d"(c), "d"(d), "l"(pol)
               : "memory");
}

// FP64 tensor-core MMA, 8x8x4 (SASS DMMA.8x8x4): C[8x8] += A[8x4] B[4x8].
// Fragment ownership (lane l): a = A[l>>2][l&3], b = B[l&3][l>>2],
// c = C[l>>2][2(l&3) + {0,1}].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Bulk prefetch of a global range into L2 (TMA engine, no completion).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// dmma with a volatile asm: keeps the x-pass / y-pass issue order (the
// compiler otherwise pairs the two dependent DMMAs of an accumulator).
__device__ __forceinline__ void dmma_ordered(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

}  // namespace gwg
