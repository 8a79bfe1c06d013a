// i8_core.cuh — shared machinery of the int8 tensor-core kernels (sm_100a):
// tile geometry, tcgen05 / TMEM / TMA primitives, the TMA producer and the
// single-thread MMA issuer of a persistent warp-specialised kernel, and the
// exact int64 recombination of seven 8-bit slice products.  Used by
// rotate_i8_kernel (rotate_i8.cuh) and linear_solve_kernel (linear_solve.cuh).
#pragma once

#include "gwg_device.cuh"

#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <utility>

#ifndef I8_PROFILE
#define I8_PROFILE 0
#endif
#ifndef I8_NO_MMA
#define I8_NO_MMA 0
#endif
#ifndef I8_EXP_A_ONCE
#define I8_EXP_A_ONCE 0
#endif
#ifndef I8_MMA_NOWAIT  // timing ablation only: the MMA issuer does not wait for operands
#define I8_MMA_NOWAIT 0
#endif
#ifndef I8_NO_TMA  // timing ablation only: stages marked full without loading them
#define I8_NO_TMA 0
#endif
// The B tile's eighth slot is never multiplied (BN <= 7 RB + 8 rows, whose
// accumulator columns the epilogues do not read): 1 = TMA boxes cover the
// seven slice slots only (single CTAs and trait pairs one 7-slot box, B pairs
// and 2 x 2 clusters 4 + 3 slots), so no zero-filled slot is written to shared
// memory; 0 = whole 8-slot boxes (the eighth zero-filled out of bounds)
#ifndef I8_SEVEN_SLOTS
#define I8_SEVEN_SLOTS 1
#endif
#ifndef I8_PREFETCH  // stages ahead the producer prefetches into L2 (B not L2-resident)
#define I8_PREFETCH 0  // measured: 4-16 stages ahead made c2 rotation 44.7 -> 72-78 ms, c4 linear 30.8 -> 41.7 ms
#endif

namespace gwg {



// Tile geometry shared by the int8 kernels: M = 128 SNPs, N = 7 slices x RB
// rows of the sliced operand (RB = 32 for the rotation, 24 or 32 for the
// linear terms of the split grid), K = 128 samples per stage.
template <int RB_, int STAGES_ = 4, int OUT_BUFS_ = 1, int EPI_WARPS_ = 8, int CLUSTER_ = 1,
          int PAIR_AXIS_ = 0, uint32_t EXTRA_ = 0, bool MMA2_ = false, bool WS_ = true>
struct I8Tile {
  // CLUSTER = 2: CTA pairs (a thread-block cluster) work on SNP tiles 2u and
  // 2u+1 against the same B rows; each CTA loads half of the B tile (4 of the
  // 8 slice slots) and multicasts it to both, halving the B operand's
  // L2->SMEM traffic (used where B dominates: large n, one trait per tile).
  static constexpr int CLUSTER = CLUSTER_;
  // PAIR_AXIS = 1 (CLUSTER = 2): the pair takes B tiles 2u and 2u+1 of the
  // same SNP tile instead, and each CTA loads half of the A tile (64 SNP
  // rows) and multicasts it — for one or two traits per tile (p >= 9), where
  // the SNP tile is re-read once per trait tile and dominates L2 traffic.
  // PAIR_AXIS = 2 (CLUSTER = 4): 2 x 2 clusters — SNP tiles 2u, 2u+1 x B
  // tiles 2v, 2v+1 (rank = SNP bit | B bit << 1).  Each CTA loads half of
  // its A tile (64 SNP rows) multicast to the CTA of the other B tile, and
  // half of its B tile (4 of the 8 slots) multicast to the CTA of the other
  // SNP tile: 8 + 16 KB issued per CTA and stage instead of 16 + 16 (B pairs)
  // or 16 + 32 (single CTAs), for the same 48 KB landing in each CTA.
  static constexpr int PAIR_AXIS = PAIR_AXIS_;
  static_assert(PAIR_AXIS == 0 || (PAIR_AXIS == 1 && CLUSTER == 2) ||
                    (PAIR_AXIS == 2 && CLUSTER == 4),
                "trait pairs need a CTA pair, 2 x 2 clusters four CTAs");
  static_assert(CLUSTER <= 2 || PAIR_AXIS == 2, "clusters of four are 2 x 2");
  // MMA2 (CLUSTER = 2, SNP-tile pairs): the pair runs ONE
  // tcgen05.mma.cta_group::2 of M = 256 issued by the even CTA.  Each CTA
  // keeps its own A tile and HALF of the B tile — 112 of the 224 slice rows
  // (the even CTA slots 0-2 and rows 0-15 of slot 3, the odd CTA rows 16-31
  // of slot 3 and slots 4-6) — and each CTA's TMEM receives its own 128 SNP
  // rows x 224 columns, in the same column order as the single-CTA MMA.  Per
  // CTA and stage, shared memory written by TMA and read by the MMA drops
  // from 16 + 28 KB to 16 + 14 KB (the single-CTA kernels' operand feed is
  // bound by shared-memory bandwidth, not by the tensor core), and the
  // smaller stages make the ring deeper.
  static constexpr bool MMA2 = MMA2_;
  // WS: the producer and MMA warps run converged and one elected lane issues
  // (see GWG_ELECT_BEGIN); otherwise one thread (lane 0) runs each loop
  static constexpr bool WS = WS_;
  static constexpr int BM = 128;          // SNPs per tile (UMMA M, TMEM lanes)
  static constexpr int RB = RB_;          // rows of the sliced operand per tile
  // Seven signed 8-bit slices (base-256 digits of a 55-bit integer, see
  // slice_basis_kernel) in eight shared-memory slots: the 3-D TMA box covers
  // whole slots, the eighth is zero-filled out of bounds and never multiplied.
  static constexpr int SLICES = 7;
  static constexpr int SLOTS = 8;
  static constexpr int BN = (SLICES * RB + 15) / 16 * 16;  // UMMA N = TMEM columns per buffer
  static constexpr int BK = 128;          // int8 K per stage = one 128B swizzle row
  static constexpr int UK = 32;           // K per tcgen05.mma (int8)
  static constexpr int STAGES = STAGES_;
  static constexpr int OUT_BUFS = OUT_BUFS_;     // staging tiles per epilogue warp
  static constexpr uint32_t A_BYTES = BM * BK;  // 16 KB
  static constexpr uint32_t B_BYTES = SLOTS * RB * BK;  // <= 32 KB of smem (slots)
  static constexpr int B_SLICES_PER_CTA = PAIR_AXIS == 1 ? SLOTS : PAIR_AXIS == 2 ? SLOTS / 2
                                                                     : SLOTS / CLUSTER;
  static constexpr uint32_t B_PART = B_BYTES / SLOTS * B_SLICES_PER_CTA;  // loaded per CTA
  static constexpr uint32_t B_SMEM = MMA2 ? SLICES * RB * BK / 2 : B_BYTES;  // B held per CTA
  static_assert(!MMA2 || (CLUSTER == 2 && PAIR_AXIS == 0 && RB == 32),
                "pair MMA: SNP-tile pairs on 32-row B tiles (112 rows = 14 swizzle atoms per CTA)");
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_SMEM;
  // bytes TMA lands in one CTA's stage (non-MMA2): the seven slice slots
  static constexpr uint32_t STAGE_TX = I8_SEVEN_SLOTS ? A_BYTES + SLICES * RB * BK : STAGE_BYTES;
  static constexpr int EPI_WARPS = EPI_WARPS_;  // multiple of 4 (TMEM lane quarters)
  static constexpr int THREADS = (4 + EPI_WARPS) * 32;  // 0 TMA, 1 MMA, 2-3 idle, 4.. epilogue
  static constexpr int TMEM_COLS = 512;   // ACC_BUFS accumulator buffers x BN
  static constexpr int ACC_BUFS = 2;      // MMA runs up to one tile ahead
  static_assert(ACC_BUFS * BN <= TMEM_COLS, "accumulator buffers fit TMEM");
  static constexpr int OUT_Q = 16;        // output box: 16 doubles (128 B) x 32 SNPs
  static constexpr uint32_t OUT_TILE = OUT_Q * 32 * 8;     // one 4 KB staging tile
  static constexpr uint32_t OUT_BYTES = OUT_BUFS * OUT_TILE;  // staging per epilogue warp
  // kernel-specific shared memory after the staging tiles (1024-aligned)
  static constexpr uint32_t EXTRA = (EXTRA_ + 15) / 16 * 16;
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * STAGE_BYTES + size_t(EPI_WARPS) * OUT_BYTES + EXTRA + 1024 + 256;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(BN % 16 == 0 && BN <= 256 && RB % 8 == 0, "UMMA N / swizzle atoms");
  static_assert(BN <= SLOTS * RB, "the MMA reads only loaded (or zero-filled) slot rows");
};
using I8Cfg = I8Tile<32>;

// ---- tcgen05 primitives --------------------------------------------------------

__device__ __forceinline__ bool lane_is_0() { return (threadIdx.x & 31) == 0; }

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

template <int BN, int BM>
__device__ __forceinline__ constexpr uint32_t i8_instr_desc() {
  // c_format S32 (2) @[4,6), a/b format signed int8 (1) @[7,10)/[10,13),
  // K-major A and B, N >> 3 @[17,23), M >> 4 @[24,29).
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
         (uint32_t(BM >> 4) << 24);
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

// 3-D TMA load multicast to the CTAs in cta_mask (same smem offset and
// mbarrier offset in each destination CTA).
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, int32_t c0,
                                               int32_t c1, int32_t c2, uint64_t* bar,
                                               uint16_t cta_mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6, %7;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
      "h"(cta_mask), "l"(policy)
      : "memory");
}

// TMA prefetch of a box into L2 (no shared-memory destination, no barrier).
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int32_t c0, int32_t c1,
                                                int32_t c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

// 2-D TMA load multicast to the CTAs in cta_mask.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int32_t c0,
                                               int32_t c1, uint64_t* bar, uint16_t cta_mask,
                                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)),
      "h"(cta_mask), "l"(policy)
      : "memory");
}

// MMA completion -> arrive on the same-offset mbarrier of every CTA in cta_mask.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// ---- CTA-pair (cta_group::2) primitives ----

__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// completion of the pair's MMAs -> arrive on the same-offset mbarrier of both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

// shared::cluster address of the same-offset location in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA loads into this CTA's shared memory completing on an mbarrier that may
// live in the peer CTA of the pair (cluster address; cta_group::2).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int32_t c0,
                                                 int32_t c1, uint32_t bar_cluster,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, int32_t c0,
                                                 int32_t c1, int32_t c2, uint32_t bar_cluster,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster),
      "l"(policy)
      : "memory");
}

// ---- warp-collective issue (the producer and MMA warps run converged) ----
// Every lane computes the same (warp-uniform) operands, so they live in
// uniform registers, and one lane chosen by elect.sync issues the
// instruction.  Measured on the B200 (tools/i8_peak.cu): a single thread
// inside a lane-0 branch issuing tcgen05.mma pays a per-instruction
// waterfall (ELECT / R2UR.BROADCAST / BRA.U.ANY) that capped an M128 N224
// K32 MMA stream with a commit per 4 MMAs at 2,932 TOP/s; the same stream
// issued warp-collectively runs at 4,439 TOP/s.  elect.sync with a full
// mask elects the same (lowest) lane every time, so a commit tracks the
// MMAs the same lane issued.  In the kernels, where operand arrival and the
// epilogue pace the MMA, the gain is smaller and not uniform (c1
// linear_solve 2.39 -> 2.35 ms, c4 30.3 -> 29.3 ms; but the rotation 0.686
// -> 0.736 ms and the cta_group::2 linear_solve at c2 18.3 -> 20.6 ms), so
// each kernel configuration chooses (I8Tile WS).
#define GWG_ELECT_BEGIN "{\n.reg .pred e_;\nelect.sync _|e_, 0xffffffff;\n"
// WS = true: the warp-collective form (elected lane); false: the plain
// instruction for a caller that is already one thread
#define GWG_ISSUE(WS, INSTR, ...)                                    \
  do {                                                               \
    if constexpr (WS)                                                \
      asm volatile(GWG_ELECT_BEGIN "@e_ " INSTR "\n}\n" __VA_ARGS__); \
    else                                                             \
      asm volatile(INSTR __VA_ARGS__);                               \
  } while (0)

// Barrier waits of the loops: every lane polls.  (Lane 0 polling and a
// __syncwarp before the elected issue measured far slower: c1 linear_solve
// 2.35 -> 3.60 ms.)
template <bool WS>
__device__ __forceinline__ void mbar_wait_w(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
}
template <bool WS>
__device__ __forceinline__ void mbar_wait_cluster_w(uint64_t* bar, uint32_t parity) {
  mbar_wait_cluster(bar, parity);
}

template <bool WS>
__device__ __forceinline__ void umma_i8_w(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  if constexpr (WS)
    asm volatile(
        GWG_ELECT_BEGIN ".reg .pred p_;\nsetp.ne.b32 p_, %4, 0;\n"
        "@e_ tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p_;\n}\n" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    umma_i8(tmem_d, a_desc, b_desc, idesc, accumulate);
}
template <bool WS>
__device__ __forceinline__ void umma_i8_pair_w(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  if constexpr (WS)
    asm volatile(
        GWG_ELECT_BEGIN ".reg .pred p_;\nsetp.ne.b32 p_, %4, 0;\n"
        "@e_ tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p_;\n}\n" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    umma_i8_pair(tmem_d, a_desc, b_desc, idesc, accumulate);
}
template <bool WS>
__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
  GWG_ISSUE(WS, "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];",
            ::"r"(smem_u32(bar))
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void umma_commit_mc_w(uint64_t* bar, uint16_t cta_mask) {
  GWG_ISSUE(WS,
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;",
            ::"r"(smem_u32(bar)), "h"(cta_mask)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void umma_commit_pair_w(uint64_t* bar) {
  GWG_ISSUE(WS,
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;",
            ::"r"(smem_u32(bar)), "h"(uint16_t(3))
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void mbar_arrive_expect_tx_w(uint64_t* bar, uint32_t bytes) {
  GWG_ISSUE(WS, "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;",
            ::"r"(smem_u32(bar)), "r"(bytes)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void mbar_arrive_w(uint64_t* bar) {
  GWG_ISSUE(WS, "mbarrier.arrive.shared::cta.b64 _, [%0];", ::"r"(smem_u32(bar)) : "memory");
}
template <bool WS>
__device__ __forceinline__ void tma_load_2d_w(void* dst, const CUtensorMap* map, int32_t c0,
                                              int32_t c1, uint64_t* bar, uint64_t policy) {
  GWG_ISSUE(WS,
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;",
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
            "r"(smem_u32(bar)), "l"(policy)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void tma_load_3d_w(void* dst, const CUtensorMap* map, int32_t c0,
                                              int32_t c1, int32_t c2, uint64_t* bar,
                                              uint64_t policy) {
  GWG_ISSUE(WS,
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;",
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
            "r"(c2), "r"(smem_u32(bar)), "l"(policy)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void tma_load_3d_mc_w(void* dst, const CUtensorMap* map, int32_t c0,
                                                 int32_t c1, int32_t c2, uint64_t* bar,
                                                 uint16_t cta_mask, uint64_t policy) {
  GWG_ISSUE(WS,
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            ".multicast::cluster.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6, %7;",
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
            "r"(c2), "r"(smem_u32(bar)), "h"(cta_mask), "l"(policy)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void tma_load_2d_mc_w(void* dst, const CUtensorMap* map, int32_t c0,
                                                 int32_t c1, uint64_t* bar, uint16_t cta_mask,
                                                 uint64_t policy) {
  GWG_ISSUE(WS,
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            ".multicast::cluster.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;",
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
            "r"(smem_u32(bar)), "h"(cta_mask), "l"(policy)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void tma_load_2d_pair_w(void* dst, const CUtensorMap* map, int32_t c0,
                                                   int32_t c1, uint32_t bar_cluster,
                                                   uint64_t policy) {
  GWG_ISSUE(WS,
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;",
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
            "r"(bar_cluster), "l"(policy)
            : "memory");
}
template <bool WS>
__device__ __forceinline__ void tma_load_3d_pair_w(void* dst, const CUtensorMap* map, int32_t c0,
                                                   int32_t c1, int32_t c2, uint32_t bar_cluster,
                                                   uint64_t policy) {
  GWG_ISSUE(WS,
            "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;",
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
            "r"(c2), "r"(bar_cluster), "l"(policy)
            : "memory");
}

// All threads of the cluster (release/acquire: barrier inits, smem writes).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 8 consecutive TMEM columns of this warp's 32 lanes into 8 registers.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}

// W consecutive TMEM columns (W = 1, 2, 4, 8) of this warp's 32 lanes.
template <int W>
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, int32_t (&v)[W]) {
  if constexpr (W == 8) {
    tmem_ld8(taddr, v);
  } else if constexpr (W == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
  } else if constexpr (W == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(v[0]), "=r"(v[1])
                 : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[0]) : "r"(taddr));
  }
}

// Exact recombination of the seven slice products of one output column.
// The sliced value is sigma 2^-55 N, N = sum_s d_s 256^(6-s) (|d_s| <= 128),
// so the column is sigma 2^-55 sum_s P_s 256^(6-s) with P_s the int32 slice
// products: hi = P0 2^16 + P1 2^8 + P2 and lo = P3 2^24 + ... + P6 are exact
// int64 (< 2^48, < 2^56); lo's bits above 2^32 move into hi (both then below
// 2^53, exactly convertible), one FMA rounds hi 2^32 + lo once, and the
// power-of-two scale sc55 = sigma 2^-55 is applied exactly.
__device__ __forceinline__ double i8_recombine(const int32_t a0, const int32_t a1, const int32_t a2,
                                               const int32_t a3, const int32_t a4, const int32_t a5,
                                               const int32_t a6, double sc55) {
  const long long hi = (long long)a0 * (1ll << 16) + (long long)a1 * (1ll << 8) + (long long)a2;
  const long long lo = (long long)a3 * (1ll << 24) + (long long)a4 * (1ll << 16) +
                       (long long)a5 * (1ll << 8) + (long long)a6;
  // lo = (lo >> 32) 2^32 + its low word (two's complement): the carry joins hi
  return fma(double(hi + (lo >> 32)), 0x1p32, double(uint32_t(lo))) * sc55;
}

// TMA 2-D store shared -> global (bulk async group of the issuing thread).
// Results stream out with an L2 evict_first hint: measured on the B200, the
// default policy made L2 fetch the written lines from HBM first (rotation:
// 0.49 GB of DRAM reads for 0.74 GB written; with the hint 0.11 GB, the
// algorithmic input bytes, and 4.5% faster).
#ifndef I8_STORE_POLICY
#define I8_STORE_POLICY 0  // 0 evict_first, 1 evict_normal, 2 evict_last
#endif
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0,
                                             int32_t c1) {
  const uint64_t pol = I8_STORE_POLICY == 1   ? policy_evict_normal()
                       : I8_STORE_POLICY == 2 ? policy_evict_last()
                                              : policy_evict_first();
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint"
      " [%0, {%1, %2}], [%3], %4;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(pol)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// at most one bulk store group of this thread still reading shared memory
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- shared pipeline: TMA producer, MMA issuer, TMEM setup ---------------------

// Shared-memory carve-up of an I8Tile kernel.
template <class C>
struct I8Smem {
  unsigned char* base;     // STAGES x (A | B), 1024-aligned for SWIZZLE_128B
  unsigned char* staging;  // [epilogue warp][OUT_BYTES]
  unsigned char* extra;    // C::EXTRA bytes for the kernel's own use
  uint64_t* full;
  uint64_t* empty;
  uint64_t* acc_full;      // [ACC_BUFS]
  uint64_t* acc_empty;     // [ACC_BUFS]
  uint32_t* tmem_slot;
  __device__ explicit I8Smem(unsigned char* raw) {
    // align by pointer arithmetic on `raw` (not through an integer cast), so
    // the compiler keeps the shared-memory provenance of every derived
    // pointer and emits LDS/STS instead of generic loads and stores
    base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    staging = base + C::STAGES * C::STAGE_BYTES;
    extra = staging + C::EPI_WARPS * C::OUT_BYTES;
    full = reinterpret_cast<uint64_t*>(extra + C::EXTRA);
    empty = full + C::STAGES;
    acc_full = empty + C::STAGES;
    acc_empty = acc_full + C::ACC_BUFS;
    tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::ACC_BUFS);
  }
};

// Barrier init + TMEM allocation (warp 1); returns the TMEM base address.
// acc_arrivals = epilogue warps that release each accumulator buffer.
template <class C>
__device__ __forceinline__ uint32_t i8_setup(const I8Smem<C>& sm, int warp,
                                             int acc_arrivals = C::EPI_WARPS) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      // the MMA of every CTA reading this stage (MMA2: the pair's one MMA)
      mbar_init(&sm.empty[s], C::MMA2 ? 1 : C::CLUSTER);
    }
    for (int b = 0; b < C::ACC_BUFS; ++b) {
      mbar_init(&sm.acc_full[b], 1);
      // one arrive per epilogue warp using it (MMA2: of both CTAs, at the even CTA)
      mbar_init(&sm.acc_empty[b], C::MMA2 ? 2 * acc_arrivals : acc_arrivals);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (C::MMA2) {  // both CTAs of the pair, collectively
      asm volatile(
          "tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
              smem_u32(sm.tmem_slot)),
          "n"(C::TMEM_COLS)
          : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile(
          "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
              smem_u32(sm.tmem_slot)),
          "n"(C::TMEM_COLS)
          : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (C::CLUSTER > 1)
    cluster_sync_all();  // the peer's barriers exist before any multicast lands
  else
    __syncthreads();
  tc_fence_after();
  return *sm.tmem_slot;
}

template <class C>
__device__ __forceinline__ void i8_teardown(uint32_t tmem_base, int warp) {
  if (C::CLUSTER > 1)
    cluster_sync_all();  // no CTA leaves while its peer may still signal its barriers
  else
    __syncthreads();
  if (warp == 1) {
    if constexpr (C::MMA2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(C::TMEM_COLS)
                   : "memory");
  }
}

// Epilogue warp: this tile's accumulator buffer may be overwritten (MMA2: the
// arrival goes to the even CTA, whose thread issues the pair's MMAs).
template <class C>
__device__ __forceinline__ void i8_acc_release(const I8Smem<C>& sm, int buf) {
  if constexpr (C::MMA2)
    mbar_arrive_cluster(mapa_u32(&sm.acc_empty[buf], 0));
  else
    mbar_arrive(&sm.acc_empty[buf]);
}

// Tile rasterisation shared by producer and epilogues: groups of I8_GROUP_M
// SNP tiles, and inside a group the SNP tile fastest, so the CTAs of one wave
// cover ~148/16 slice-row tiles x 16 SNP tiles: both operands' working sets
// stay in L2 even when they do not fit whole (n = 10,000: X int8 1 GB, Z
// slices 0.8 GB, W slices 0.3 GB), and each B tile is fetched from HBM once
// per group instead of once per SNP tile.
#ifndef I8_GROUP
#define I8_GROUP 16
#endif
constexpr int I8_GROUP_M = I8_GROUP;
__device__ __forceinline__ void i8_tile_coords(int tile, int tiles_m, int tiles_r, int& tm,
                                               int& tr) {
  const int per_group = I8_GROUP_M * tiles_r;
  const int grp = tile / per_group;
  const int rem = tile - grp * per_group;
  const int rows = min(I8_GROUP_M, tiles_m - grp * I8_GROUP_M);
  tr = rem / rows;
  tm = grp * I8_GROUP_M + (rem - tr * rows);
}

// Persistent static schedule over scheduling units (one CTA, or one CTA pair
// for CLUSTER = 2: the pair takes SNP tiles 2u and 2u+1 of one B tile).
// raster = 1: the B-tile index fastest over the whole grid instead — the 148
// tiles in flight then cover one or two SNP tiles x every B tile, so results
// in numpy order (SNP-major rows of t*p doubles) are written as a few
// contiguous megabytes instead of thousands of scattered 256-byte pieces
// (B must then stay L2-resident: the W slices of every trait)
template <class C>
struct I8Sched {
  int rank, unit, units, tm_units, tiles_r, my_tiles, raster;
  __device__ I8Sched(int tiles_m, int tiles_r_, int raster_ = 0) : tiles_r(tiles_r_), raster(raster_) {
    rank = C::CLUSTER > 1 ? int(blockIdx.x % C::CLUSTER) : 0;
    unit = int(blockIdx.x / C::CLUSTER);
    units = int(gridDim.x / C::CLUSTER);
    // unit grid: (SNP-tile pairs x B tiles), (SNP tiles x B-tile pairs) or,
    // for 2 x 2 clusters, (SNP-tile pairs x B-tile pairs)
    tm_units = C::PAIR_AXIS == 1 ? tiles_m : (tiles_m + 1) / (C::CLUSTER > 1 ? 2 : 1);
    tr_units = C::PAIR_AXIS ? (tiles_r + 1) / 2 : tiles_r;
    const int ntiles = tm_units * tr_units;
    my_tiles = unit < ntiles ? (ntiles - 1 - unit) / units + 1 : 0;
  }
  int tr_units;
  __device__ void coords(int lt, int& tm, int& tr) const {
    int tu, ru;
    if (raster) {
      const int idx = unit + lt * units;
      tu = idx / tr_units;
      ru = idx - tu * tr_units;
    } else {
      i8_tile_coords(unit + lt * units, tm_units, tr_units, tu, ru);
    }
    if constexpr (C::PAIR_AXIS == 2) {
      tm = tu * 2 + (rank & 1);
      tr = ru * 2 + (rank >> 1);
    } else {
      tm = C::PAIR_AXIS ? tu : tu * C::CLUSTER + rank;
      tr = C::PAIR_AXIS ? ru * 2 + rank : ru;
    }
  }
};

// Warp 0, all lanes converged (one elected lane issues): A = int8 SNP tile (box 128 k x 128 SNPs), B = RB rows
// of all 8 slices (box 128 k x RB x 8).  Tiles: i8_tile_coords (the rows
// of the sliced operand fastest, so the SNP tile is reused from L2).
// MMA2: tmap_bh is the half-slot map (box 128 k x 16 rows x 1 slot) for the
// B rows split between the two CTAs.
template <class C>
__device__ __forceinline__ void i8_produce(const I8Smem<C>& sm, const CUtensorMap* tmap_x,
                                           const CUtensorMap* tmap_b, const I8Sched<C>& sch,
                                           int kstages, bool b_resident,
                                           const CUtensorMap* tmap_bh = nullptr) {
  // B small enough to stay in L2 for the whole launch: keep it (evict_last).
  // A (the int8 SNP tile) is re-read by every B tile of its group, so it is
  // NOT evict_first (measured: linear_solve DRAM reads 2.66 -> 1.61 GB, 2.84
  // -> 2.70 ms at c1); the results stream out evict_first (tma_store_2d).
#ifndef I8_X_POLICY  // L2 policy of the SNP-tile loads: 0 evict_normal, 1 evict_last
#define I8_X_POLICY 0
#endif
  const uint64_t pol_x = I8_X_POLICY == 1 ? policy_evict_last() : policy_evict_normal();
  const uint64_t pol_b = b_resident ? policy_evict_last() : policy_evict_normal();
  // B streaming from HBM (large n): prefetch the operand boxes of the stage
  // I8_PREFETCH stages ahead into L2, so the stage ring (4 x 48 KB, ~1,800 MMA
  // cycles) only has to cover L2 latency, not HBM latency
  const int pf = b_resident ? 0 : I8_PREFETCH;
  const int total = sch.my_tiles * kstages;
  int g = 0;
#if I8_PROFILE
  long long t_empty = 0, t0 = clock64();
#endif
  for (int lt = 0; lt < sch.my_tiles; ++lt) {
    int tm, tr;
    sch.coords(lt, tm, tr);
    for (int ks = 0; ks < kstages; ++ks, ++g) {
      const int s = g % C::STAGES;
      // CLUSTER = 2: empty[s] completes only when BOTH CTAs' MMAs are done with
      // stage s, since this CTA's multicast also writes the peer's stage
#if I8_PROFILE
      long long te = clock64();
#endif
      if (g >= C::STAGES) mbar_wait_w<C::WS>(&sm.empty[s], ((g / C::STAGES) - 1) & 1);
#if I8_PROFILE
      t_empty += clock64() - te;
#endif
      unsigned char* st = sm.base + s * C::STAGE_BYTES;
      if (I8_NO_TMA) {
        if (!C::MMA2 || sch.rank == 0) mbar_arrive_w<C::WS>(&sm.full[s]);
        continue;
      }
      if constexpr (C::MMA2) {
        // both CTAs' loads complete on the even CTA's full[s], which expects
        // the pair's bytes (a peer transfer landing first only drives the
        // transaction count negative until then)
        if (sch.rank == 0) mbar_arrive_expect_tx_w<C::WS>(&sm.full[s], 2 * C::STAGE_BYTES);
        const uint32_t fb = mapa_u32(&sm.full[s], 0);
        tma_load_2d_pair_w<C::WS>(st, tmap_x, ks * C::BK, tm * C::BM, fb, pol_x);
        unsigned char* sb = st + C::A_BYTES;
        const int r0 = tr * C::RB;
        constexpr int H = C::RB / 2;
        if (sch.rank == 0) {  // B rows 0-111: slots 0-2, slot 3 rows 0-15
          tma_load_3d_pair_w<C::WS>(sb, tmap_b, ks * C::BK, r0, 0, fb, pol_b);
          tma_load_3d_pair_w<C::WS>(sb + 3 * C::RB * C::BK, tmap_bh, ks * C::BK, r0, 3, fb, pol_b);
        } else {              // B rows 112-223: slot 3 rows 16-31, slots 4-6
          tma_load_3d_pair_w<C::WS>(sb, tmap_bh, ks * C::BK, r0 + H, 3, fb, pol_b);
          tma_load_3d_pair_w<C::WS>(sb + H * C::BK, tmap_b, ks * C::BK, r0, 4, fb, pol_b);
        }
        continue;
      }
      if (pf && g + pf < total) {
        const int gf = g + pf, ltf = gf / kstages, ksf = gf - ltf * kstages;
        int tmf, trf;
        sch.coords(ltf, tmf, trf);
        if (C::PAIR_AXIS == 1) {
          if (lane_is_0()) tma_prefetch_3d(tmap_b, ksf * C::BK, trf * C::RB, 0);
        } else {
          if (lane_is_0()) tma_prefetch_2d(tmap_x, ksf * C::BK, tmf * C::BM);
          if (lane_is_0()) tma_prefetch_3d(tmap_b, ksf * C::BK, trf * C::RB, sch.rank * C::B_SLICES_PER_CTA);
        }
      }
      // timing probe only (I8_EXP_A_ONCE): the A box of the first K stage
      // only, the rest left stale — how much the kernel gains without the
      // per-stage SNP-tile ingress
      const bool a_skip = I8_EXP_A_ONCE == 1 && C::PAIR_AXIS == 0 && (g % C::STAGES) != 0;
      const bool b_skip = I8_EXP_A_ONCE == 2 && C::PAIR_AXIS == 0 && (g % C::STAGES) != 0;
      mbar_arrive_expect_tx_w<C::WS>(&sm.full[s], a_skip ? C::STAGE_TX - C::A_BYTES
                                                  : b_skip ? C::A_BYTES : C::STAGE_TX);
      if (b_skip) {
        tma_load_2d_w<C::WS>(st, tmap_x, ks * C::BK, tm * C::BM, &sm.full[s], pol_x);
        continue;
      }
      if constexpr (C::PAIR_AXIS == 2) {
        // 2 x 2: A rows [rb * 64, +64) to both CTAs of this SNP tile (ranks
        // sb, sb + 2), B slots [sb * 4, +4) to both CTAs of this B tile
        // (ranks 2 rb, 2 rb + 1); partial tiles past either edge still load
        // (zero-filled) boxes so every barrier completes
        const int sb = sch.rank & 1, rb = sch.rank >> 1;
        tma_load_2d_mc_w<C::WS>(st + rb * (C::A_BYTES / 2), tmap_x, ks * C::BK,
                                tm * C::BM + rb * (C::BM / 2), &sm.full[s],
                                uint16_t((1u << sb) | (1u << (sb + 2))), pol_x);
        tma_load_3d_mc_w<C::WS>(st + C::A_BYTES + sb * C::B_PART, sb ? tmap_bh : tmap_b,
                                ks * C::BK, tr * C::RB,
                                sb * C::B_SLICES_PER_CTA, &sm.full[s], uint16_t(3u << (2 * rb)),
                                pol_b);
        continue;
      }
      if constexpr (C::PAIR_AXIS == 1) {
        // half of the shared SNP tile each (box 128 k x 64 SNPs), multicast;
        // this CTA's own B tile, all 8 slots
        tma_load_2d_mc_w<C::WS>(st + sch.rank * (C::A_BYTES / 2), tmap_x, ks * C::BK,
                       tm * C::BM + sch.rank * (C::BM / 2), &sm.full[s], 3, pol_x);
        tma_load_3d_w<C::WS>(st + C::A_BYTES, tmap_b, ks * C::BK, tr * C::RB, 0, &sm.full[s], pol_b);
        continue;
      }
      if (!a_skip) tma_load_2d_w<C::WS>(st, tmap_x, ks * C::BK, tm * C::BM, &sm.full[s], pol_x);
      if (C::CLUSTER > 1)
        tma_load_3d_mc_w<C::WS>(st + C::A_BYTES + sch.rank * C::B_PART,
                                sch.rank ? tmap_bh : tmap_b, ks * C::BK, tr * C::RB,
                       sch.rank * C::B_SLICES_PER_CTA, &sm.full[s],
                       uint16_t((1u << C::CLUSTER) - 1), pol_b);
      else
        tma_load_3d_w<C::WS>(st + C::A_BYTES, tmap_b, ks * C::BK, tr * C::RB, 0, &sm.full[s], pol_b);
    }
  }
#if I8_PROFILE
  if (blockIdx.x < 4 && lane_is_0())
    printf("I8PROF producer cta %d total %lld wait_empty %lld\n", int(blockIdx.x), clock64() - t0,
           t_empty);
#endif
}

// MMA2, even CTA only: one M = 256 tcgen05.mma.cta_group::2 per K step (its
// 128 SNP rows and half of B here, the peer's at the same shared-memory
// offsets), committed to both CTAs' barriers.
template <class C>
__device__ __forceinline__ void i8_mma_pair(const I8Smem<C>& sm, uint32_t tmem_base,
                                            int my_tiles, int kstages) {
  constexpr uint32_t idesc = i8_instr_desc<C::BN, 2 * C::BM>();
  int g = 0;
  for (int lt = 0; lt < my_tiles; ++lt) {
    const int buf = lt % C::ACC_BUFS;
    if (lt >= C::ACC_BUFS)
      mbar_wait_cluster_w<C::WS>(&sm.acc_empty[buf], ((lt / C::ACC_BUFS) - 1) & 1);
    tc_fence_after();
    const uint32_t tmem_d = tmem_base + uint32_t(buf * C::BN);
    for (int ks = 0; ks < kstages; ++ks, ++g) {
      const int s = g % C::STAGES;
      mbar_wait_w<C::WS>(&sm.full[s], (g / C::STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(sm.base + s * C::STAGE_BYTES);
      const uint32_t sb = sa + C::A_BYTES;
#if !I8_NO_MMA
#pragma unroll
      for (int k = 0; k < C::BK / C::UK; ++k)
        umma_i8_pair_w<C::WS>(tmem_d, umma_desc_sw128(sa + k * C::UK), umma_desc_sw128(sb + k * C::UK),
                     idesc, (ks | k) != 0);
#endif
      umma_commit_pair_w<C::WS>(&sm.empty[s]);  // frees stage s in both CTAs
    }
    umma_commit_pair_w<C::WS>(&sm.acc_full[buf]);  // both CTAs' accumulators ready
  }
}

// Warp 1, all lanes converged (one elected lane issues): BK/UK tcgen05.mma per
// stage into the tile's TMEM buffer.
template <class C>
__device__ __forceinline__ void i8_mma(const I8Smem<C>& sm, uint32_t tmem_base, int my_tiles,
                                       int kstages) {
  if constexpr (C::MMA2) {
    if (blockIdx.x % 2 == 0) i8_mma_pair<C>(sm, tmem_base, my_tiles, kstages);
    return;
  }
  constexpr uint16_t mask = uint16_t((1u << C::CLUSTER) - 1);
  constexpr uint32_t idesc = i8_instr_desc<C::BN, C::BM>();
  int g = 0;
#if I8_PROFILE
  long long t_acc = 0, t_full = 0, t0 = clock64();
#endif
  for (int lt = 0; lt < my_tiles; ++lt) {
    const int buf = lt % C::ACC_BUFS;
#if I8_PROFILE
    long long ta = clock64();
#endif
    if (lt >= C::ACC_BUFS) mbar_wait_w<C::WS>(&sm.acc_empty[buf], ((lt / C::ACC_BUFS) - 1) & 1);
#if I8_PROFILE
    t_acc += clock64() - ta;
#endif
    tc_fence_after();
    const uint32_t tmem_d = tmem_base + uint32_t(buf * C::BN);
    for (int ks = 0; ks < kstages; ++ks, ++g) {
      const int s = g % C::STAGES;
#if I8_PROFILE
      long long tf = clock64();
#endif
      if (!I8_MMA_NOWAIT) mbar_wait_w<C::WS>(&sm.full[s], (g / C::STAGES) & 1);
#if I8_PROFILE
      t_full += clock64() - tf;
#endif
      tc_fence_after();
      const uint32_t sa = smem_u32(sm.base + s * C::STAGE_BYTES);
      const uint32_t sb = sa + C::A_BYTES;
#if !I8_NO_MMA  // timing ablation only: the barrier protocol without the MMAs
#pragma unroll
      for (int k = 0; k < C::BK / C::UK; ++k)
        umma_i8_w<C::WS>(tmem_d, umma_desc_sw128(sa + k * C::UK), umma_desc_sw128(sb + k * C::UK), idesc,
                (ks | k) != 0);
#endif
      // frees the smem stage (in every CTA of the pair) when these MMAs finish
      if (C::CLUSTER > 1)
        umma_commit_mc_w<C::WS>(&sm.empty[s], mask);
      else
        umma_commit_w<C::WS>(&sm.empty[s]);
    }
    umma_commit_w<C::WS>(&sm.acc_full[buf]);  // accumulator ready for the epilogue
  }
#if I8_PROFILE
  if (blockIdx.x < 4 && lane_is_0())
    printf("I8PROF mma cta %d tiles %d total %lld wait_acc_empty %lld wait_full %lld\n",
           int(blockIdx.x), my_tiles, clock64() - t0, t_acc, t_full);
#endif
}

// Host: launch an I8Tile kernel over `units` scheduling units (CTA pairs for
// CLUSTER = 2) with at most `sms` CTAs, in clusters of C::CLUSTER CTAs.
template <class C, typename... KArgs, typename... Args>
cudaError_t i8_launch(void (*kern)(KArgs...), int64_t units, int sms, cudaStream_t s,
                      Args&&... args) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(C::SMEM_BYTES));
  if (e != cudaSuccess) return e;
  int64_t max_units = sms / C::CLUSTER;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CLUSTER;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (C::CLUSTER > 2) {
    // clusters of four need four free SMs in one GPC: launch only as many
    // as can be co-resident (a persistent static schedule must not leave a
    // second wave), once per kernel (the answer depends on the device only)
    static int resident = 0;
    if (resident == 0) {
      cfg.gridDim = dim3(unsigned(max_units * C::CLUSTER));
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
        (void)cudaGetLastError();
        n = int(max_units);
      }
      resident = n;
    }
    max_units = std::min<int64_t>(max_units, resident);
  }
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, max_units))) * C::CLUSTER;
  cfg.gridDim = dim3(unsigned(grid));
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace gwg
