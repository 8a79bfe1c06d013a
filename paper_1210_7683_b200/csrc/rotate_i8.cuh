// rotate_i8.cuh — exact-integer rotation of genotype-coded SNP slabs on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators).
//
// X' = Z^T X_R where X_R holds integer genotype codes (BASELINE.json: {0,1,2}).
// Each eigenvector z_r (column r of Z) is scaled by a power of two sigma_r
// (|z_r / sigma_r| <= 1/2) and split into eight 7-bit signed slices,
//     z_r / sigma_r = sum_{s<8} q_{s,r} 2^{-7(s+1)} + O(2^{-57}),  |q| <= 64,
// so  X'[r, i] = sigma_r sum_s 2^{-7(s+1)} (q_{s,r} . x_i)  where every inner
// product is an EXACT int32 dot product of int8 vectors (|q x| <= 64*127, so
// exact for n < 262,000).  The eight partial results are combined in FP64 in a
// fixed order (s = 7 .. 0): the rotation error is ~1 ulp, below a DGEMM's, and
// each column depends only on (Z, x_i) — bitwise identical for any slab
// width, like rotate_kernel.  The DMMA rotation (rotate_kernel.cuh) remains the
// general path for real-valued SNP data.
//
// GEMM view per CTA tile: M = 128 SNPs (A = X int8, K-major), N = 256 =
// 8 slices x 32 eigen-rows (B = slices, K-major), K = samples, int32 D in TMEM.
// Warp roles: warp 0 = TMA producer (SWIZZLE_128B boxes, 4-stage mbarrier
// ring), warp 1 = MMA issuer (one thread, 4 x tcgen05.mma M128 N256 K32 per
// stage) and TMEM owner (2 x 256 columns: double-buffered accumulators),
// warps 4-7 = epilogue (tcgen05.ld 32x32b, FP64 recombination, stores of X'
// and X'.X').
#pragma once

#include "gwg_device.cuh"

namespace gwg {

struct I8Cfg {
  static constexpr int BM = 128;          // SNPs per tile (UMMA M, TMEM lanes)
  static constexpr int RB = 32;           // eigen-rows per tile
  static constexpr int SLICES = 8;
  static constexpr int BN = SLICES * RB;  // 256 = UMMA N
  static constexpr int BK = 128;          // int8 K per stage = one 128B swizzle row
  static constexpr int UK = 32;           // K per tcgen05.mma (int8)
  static constexpr int STAGES = 4;
  static constexpr uint32_t A_BYTES = BM * BK;  // 16 KB
  static constexpr uint32_t B_BYTES = BN * BK;  // 32 KB
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int THREADS = 256;     // 8 warps: 0 TMA, 1 MMA, 4..7 epilogue
  static constexpr int TMEM_COLS = 512;   // 2 accumulator buffers x 256
  static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 + 256;
};

struct I8Args {
  double* dst;          // X' (n x cols, ld ldd)
  double* dst_sq;       // X'.X' (same layout)
  const double* scale;  // sigma_r per eigen-row (n)
  int64_t ldd;
  int32_t n;
  int32_t cols;
  int32_t tiles_m;      // ceil(cols / 128)
  int32_t tiles_r;      // ceil(n / 32)
  int32_t kstages;      // kp / 128
};

// ---- tcgen05 primitives --------------------------------------------------------

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  // K-major SWIZZLE_128B canonical layout: 8-row x 128B atoms, SBO = 1024 B,
  // LBO unused (1), version 1 (sm_100), layout type 2 (SWIZZLE_128B).
  uint64_t d = 0;
  d |= uint64_t((smem_addr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;                   // LBO (ignored for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;           // SBO
  d |= uint64_t(1) << 46;                   // version
  d |= uint64_t(2) << 61;                   // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ constexpr uint32_t i8_instr_desc() {
  // c_format S32 (2) @[4,6), a/b format signed int8 (1) @[7,10)/[10,13),
  // K-major A and B, N >> 3 @[17,23), M >> 4 @[24,29).
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(I8Cfg::BN >> 3) << 17) |
         (uint32_t(I8Cfg::BM >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, int32_t c2, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
      "l"(policy)
      : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes into 32 registers.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
}

// 16 consecutive TMEM columns of this warp's 32 lanes into 16 registers.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- the kernel ----------------------------------------------------------------

__global__ void __launch_bounds__(I8Cfg::THREADS, 1)
    rotate_i8_kernel(const __grid_constant__ CUtensorMap tmap_x,
                     const __grid_constant__ CUtensorMap tmap_z, const I8Args a) {
  using C = I8Cfg;
  extern __shared__ __align__(1024) unsigned char smem_i8[];
  // stages must be 1024-aligned for SWIZZLE_128B
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_i8) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_r;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM allocation (whole warp), address to smem
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            smem_u32(tmem_slot)),
        "n"(C::TMEM_COLS)
        : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      const uint64_t pol_x = policy_evict_first();
      const uint64_t pol_z = policy_evict_last();
      int g = 0;
      for (int lt = 0; lt < my_tiles; ++lt) {
        const int tile = blockIdx.x + lt * gridDim.x;
        const int tm = tile / a.tiles_r;   // SNP tile (r-blocks fastest: X tile reused)
        const int tr = tile - tm * a.tiles_r;
        for (int ks = 0; ks < a.kstages; ++ks, ++g) {
          const int s = g % C::STAGES;
          if (g >= C::STAGES) mbar_wait(&empty[s], ((g / C::STAGES) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          unsigned char* st = base + s * C::STAGE_BYTES;
          tma_load_2d(st, &tmap_x, ks * C::BK, tm * C::BM, &full[s], pol_x);
          tma_load_3d(st + C::A_BYTES, &tmap_z, ks * C::BK, tr * C::RB, 0, &full[s], pol_z);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = i8_instr_desc();
      int g = 0;
      for (int lt = 0; lt < my_tiles; ++lt) {
        const int buf = lt & 1;
        if (lt >= 2) mbar_wait(&acc_empty[buf], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(buf * C::BN);
        for (int ks = 0; ks < a.kstages; ++ks, ++g) {
          const int s = g % C::STAGES;
          mbar_wait(&full[s], (g / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(base + s * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / C::UK; ++k)
            umma_i8(tmem_d, umma_desc_sw128(sa + k * C::UK), umma_desc_sw128(sb + k * C::UK),
                    idesc, (ks | k) != 0);
          umma_commit(&empty[s]);  // frees the smem stage when these MMAs finish
        }
        umma_commit(&acc_full[buf]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: warp (w % 4) owns TMEM lanes 32*(w%4).. ----
    const int q = warp & 3;
    for (int lt = 0; lt < my_tiles; ++lt) {
      const int buf = lt & 1;
      const int tile = blockIdx.x + lt * gridDim.x;
      const int tm = tile / a.tiles_r;
      const int tr = tile - tm * a.tiles_r;
      mbar_wait(&acc_full[buf], (lt >> 1) & 1);
      tc_fence_after();
      const int i = tm * C::BM + q * 32 + lane;   // SNP column of this thread's lane
      const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(buf * C::BN);
      const bool valid = i < a.cols;
      double* d = a.dst + int64_t(valid ? i : 0) * a.ldd;
      double* d2 = a.dst_sq + int64_t(valid ? i : 0) * a.ldd;
#pragma unroll
      for (int h = 0; h < C::RB / 16; ++h) {  // 16 eigen-rows at a time
        double outv[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) outv[r] = 0.0;
        // slices from least to most significant: fixed summation order
#pragma unroll
        for (int s = C::SLICES - 1; s >= 0; --s) {
          int32_t v[16];
          tmem_ld16(taddr + uint32_t(s * C::RB + h * 16), v);
          tmem_ld_wait();
          const double w = ldexp(1.0, -7 * (s + 1));
#pragma unroll
          for (int r = 0; r < 16; ++r) outv[r] = fma(double(v[r]), w, outv[r]);
        }
        if (valid) {
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const int row = tr * C::RB + h * 16 + r;
            if (row < a.n) {
              const double x = outv[r] * __ldg(a.scale + row);
              d[row] = x;
              if (d2) d2[row] = x * x;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(C::TMEM_COLS)
                 : "memory");
}

// ---- slab / basis preparation ------------------------------------------------------

// X (n x cols, ld lds, f64 genotype codes) -> int8 [col][kp] with zero padding;
// flags (*bad = 0) any value that is not an integer in [-127, 127].
__global__ void snp_to_i8_kernel(const double* __restrict__ x, int64_t lds, int32_t n,
                                 int32_t cols, int32_t kp, int8_t* __restrict__ out,
                                 unsigned long long* __restrict__ bad) {
  const int64_t total = int64_t(cols) * kp;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = idx / kp;
    const int k = int(idx - c * kp);
    int8_t q = 0;
    if (k < n) {
      const double v = x[c * lds + k];
      if (!(v == rint(v)) || !(fabs(v) <= 127.0)) {
        *bad = 0;  // error words are reset to all ones
      } else {
        q = int8_t(v);
      }
    }
    out[idx] = q;
  }
}

// Z (n x n, ld ldz) -> slices [s][r][kp] int8 and scale[r] = sigma_r: one
// block per eigen-row r (= column r of Z).
__global__ void slice_basis_kernel(const double* __restrict__ z, int64_t ldz, int32_t n,
                                   int32_t kp, int8_t* __restrict__ slices,
                                   double* __restrict__ scale) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  const double* col = z + int64_t(r) * ldz;
  double mx = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, fabs(col[k]));
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    // sigma = 2^(e+1) with m <= 2^e, so |z / sigma| <= 1/2
    int e = 0;
    frexp(m > 0.0 ? m : 1.0, &e);  // m = f 2^e, f in [0.5, 1)
    red[0] = ldexp(1.0, e + 1);
    scale[r] = red[0];
  }
  __syncthreads();
  const double inv = 1.0 / red[0];  // exact: power of two
  const int64_t plane = int64_t(n) * kp;
  for (int k = threadIdx.x; k < kp; k += blockDim.x) {
    double v = k < n ? col[k] * inv : 0.0;  // exact scaling
#pragma unroll
    for (int s = 0; s < I8Cfg::SLICES; ++s) {
      const double t = v * 128.0;          // exact
      const double qd = rint(t);
      slices[s * plane + int64_t(r) * kp + k] = int8_t(qd);
      v = t - qd;                          // exact (Sterbenz), |v| <= 1/2
    }
  }
}

}  // namespace gwg
