// grid_split.cuh — the GLS grid for genotype-coded SNPs, split by tensor pipe.
//
// Same cells as grid_kernel.cuh (compute_tile -> solve_gls_cell,
// proj/src/grid.cpp:191-273, proj/src/gls.cpp:105-132), regrouped so that the
// SNP operand of the p linear terms stays integer:
//     S_BL[i,j,c] = X'_i^T (D_j.X_L'_c) = x_i^T W_{j,c},  W_{j,c} = Z (D_j.X_L'_c)
//     b_B[i,j]    = X'_i^T (D_j.Y'_j)   = x_i^T W_{j,p-1}, W_{j,p-1} = Z (D_j.Y'_j)
//     S_BR[i,j]   = (X'_i.X'_i)^T D_j                       (quadratic in x_i)
// Launches per slab:
//   gls_sbr_kernel (this file), a DMMA.8x8x4 GEMM: S_BR = (X'.X')^T D
//       directly (2n flop per cell), or — the default — twice, through the
//       positive exponential-sum factorisation D = E F (expsum.cpp):
//       G = (X'.X')^T E stored [SNP][r] (rowmajor), then S_BR = G F, 2r(n+t)
//       flop per SNP; S_BR is stored [trait][SNP].
//   linear_solve_kernel<P> (linear_solve.cuh): x_i^T W exactly on the int8
//       tensor cores against seven signed 8-bit slices of W (tcgen05.mma kind::i8,
//       TMEM accumulators, exact int64 recombination), and in the same
//       epilogue the bordered Cholesky solve against S_BR and the per-trait
//       context (solve_cell), b_ij out by TMA store.  The FP64 pipe is idle
//       in that kernel, so the solve costs no DMMA cycles.
//
// gls_sbr_kernel: persistent, two ping-pong consumer groups of 4 warps (one
// warp of each per SM sub-partition) half a tile out of phase, one TMA
// producer warp per group.  Warp tile (8*WO SNPs) x (8*TW traits), one DMMA
// accumulator pair per 8x8 block.  Stages: X'.X' by TMA 2-D boxes (8 k x BM
// SNPs per k-octet, zero fill past n and m) + one bulk copy of the D panel
// ([tile][k/8][trait octet][trait%8][k%8], the smem order).  Reduction order
// over k is fixed, so results stay bitwise independent of slab geometry.
#pragma once

#include "gwg_device.cuh"

namespace gwg {

template <int WO_, int TW_, int WARPS_M_, int WARPS_T_, int BK_, int STAGES_>
struct SbrCfg {
  static constexpr int WO = WO_;  // SNP octets per warp
  static constexpr int TW = TW_;  // trait octets per warp
  static constexpr int WARPS_M = WARPS_M_;
  static constexpr int WARPS_T = WARPS_T_;
  static constexpr int BK = BK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int GROUPS = 2;
  static constexpr int GWARPS = WARPS_M * WARPS_T;
  static constexpr int WARPS = GWARPS * GROUPS;
  static constexpr int THREADS = (WARPS + GROUPS) * 32;
  static constexpr int BM = 8 * WO * WARPS_M;
  static constexpr int BT = 8 * TW * WARPS_T;
  static constexpr int A_STAGE = BK * BM;  // doubles
  static constexpr int B_STAGE = BK * BT;  // doubles
  static constexpr uint32_t A_BYTES = A_STAGE * 8;
  static constexpr uint32_t B_BYTES = B_STAGE * 8;
  static constexpr size_t SMEM_BYTES =
      size_t(GROUPS) * (size_t(STAGES) * (A_BYTES + B_BYTES) + 2 * STAGES * sizeof(uint64_t)) +
      sizeof(uint64_t);
  static_assert(GWARPS == 4, "one warp of each group per SM sub-partition");
  static_assert(BK % 8 == 0 && BM <= 256, "TMA box");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

// The shipped configuration: group tile 64 SNPs x 64 traits, warp tile 32 x 32.
using SbrDefault = SbrCfg<4, 4, 2, 2, 32, 3>;

struct SbrArgs {
  const double* dpanel;  // D panels, [tile][k/8][trait octet][trait%8][k%8]
  double* sbr;           // S_BR[j * ld + i]
  int64_t ld;
  int64_t rows;
  int32_t t;
  int32_t tiles_m;
  int32_t tiles_t;
  int32_t kchunks;
  int64_t np;        // K extent of one D panel (its stride between trait tiles)
  int32_t rowmajor;  // 1: store out[i * ld + j] instead (j < t, t a multiple of BT)
  // split K: every output tile is computed as ksplit partial products over
  // kchunks / ksplit consecutive k-chunks each, partial s stored at
  // sbr + s * split_stride (summed in a fixed order by sum_partials_kernel)
  int32_t ksplit = 1;
  int64_t split_stride = 0;
  const unsigned long long* gate = nullptr;  // GWG_SNP_AUTO path gate (gate_closed)
  int32_t gate_codes = 0;
};

template <class Cfg>
__device__ __forceinline__ void sbr_issue(const CUtensorMap* tmap_q, const SbrArgs& args,
                                          double* sA, double* sB, uint64_t* full,
                                          uint64_t* empty, int g, int group, uint64_t pol_a,
                                          uint64_t pol_b) {
  constexpr int KO = Cfg::BK / 8;
  const int s = g % Cfg::STAGES;
  const int use = g / Cfg::STAGES;
  if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
  const int kc_per = args.kchunks / args.ksplit;
  const int local_tile = g / kc_per;
  const int vt = (blockIdx.x + local_tile * gridDim.x) * Cfg::GROUPS + group;
  const int tile = vt / args.ksplit;
  const int kc = (g - local_tile * kc_per) + (vt - tile * args.ksplit) * kc_per;
  const int tm = tile / args.tiles_t;
  const int tt = tile - tm * args.tiles_t;
  mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
  double* a_dst = sA + s * Cfg::A_STAGE;
#pragma unroll
  for (int ko = 0; ko < KO; ++ko)
    tma_load_2d(a_dst + ko * Cfg::BM * 8, tmap_q, (kc * KO + ko) * 8, tm * Cfg::BM, &full[s],
                pol_a);
  const double* bsrc =
      args.dpanel + size_t(tt) * size_t(args.np) * Cfg::BT + size_t(kc) * Cfg::B_STAGE;
  bulk_load(sB + s * Cfg::B_STAGE, bsrc, Cfg::B_BYTES, &full[s], pol_b);
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    gls_sbr_kernel(const __grid_constant__ CUtensorMap tmap_q, const SbrArgs args) {
  if (gate_closed(args.gate, args.gate_codes)) return;
  constexpr int KO = Cfg::BK / 8;
  constexpr int WO = Cfg::WO;
  constexpr int TW = Cfg::TW;
  constexpr int G = Cfg::GROUPS;
  extern __shared__ __align__(1024) double smem[];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool is_producer_warp = warp >= Cfg::WARPS;
  const int group = is_producer_warp ? warp - Cfg::WARPS : (warp / 4) % G;
  const int lw = (warp % 4) + 4 * (warp / (4 * G));

  double* sA = smem + size_t(group) * Cfg::STAGES * (Cfg::A_STAGE + Cfg::B_STAGE);
  double* sB = sA + Cfg::STAGES * Cfg::A_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      smem + size_t(G) * Cfg::STAGES * (Cfg::A_STAGE + Cfg::B_STAGE));
  uint64_t* full = bars + group * 2 * Cfg::STAGES;
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* go = bars + G * 2 * Cfg::STAGES;

  const int ntiles = args.tiles_m * args.tiles_t * args.ksplit;  // (tile, k-split) units
  const int kc_per = args.kchunks / args.ksplit;
  const int nsuper = (ntiles + G - 1) / G;
  const int my_super = blockIdx.x < nsuper ? (nsuper - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  int my_tiles = my_super;
  if (my_super > 0 && (blockIdx.x + (my_super - 1) * gridDim.x) * G + group >= ntiles) --my_tiles;
  const int total_iters = my_tiles * kc_per;

  if (threadIdx.x == 0) {
    for (int q = 0; q < G * 2 * Cfg::STAGES; q += 2 * Cfg::STAGES)
      for (int s = 0; s < Cfg::STAGES; ++s) {
        mbar_init(&bars[q + s], 1);
        mbar_init(&bars[q + Cfg::STAGES + s], Cfg::GWARPS);
      }
    mbar_init(go, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (is_producer_warp) {
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_normal();  // SNP tile: re-read across trait tiles
      const uint64_t pol_b = policy_evict_last();    // D panels: L2-resident
      for (int g = 0; g < total_iters; ++g)
        sbr_issue<Cfg>(&tmap_q, args, sA, sB, full, empty, g, group, pol_a, pol_b);
    }
    return;
  }

  const int wm = lw % Cfg::WARPS_M;
  const int wt = lw / Cfg::WARPS_M;
  const int half = kc_per / 2;
  if (group > 0 && my_tiles > 0) mbar_wait(go, 0);  // start half a tile late
  if (group == 0 && lw == 0 && lane == 0 && my_tiles == 0) mbar_arrive(go);
  int g = 0;
  for (int lt = 0; lt < my_tiles; ++lt) {
    const int vt = (blockIdx.x + lt * gridDim.x) * G + group;
    const int tile = vt / args.ksplit;
    double* const out = args.sbr + int64_t(vt - tile * args.ksplit) * args.split_stride;
    const int tm = tile / args.tiles_t;
    const int tt = tile - tm * args.tiles_t;

    double acc[WO][TW][2];
#pragma unroll
    for (int o = 0; o < WO; ++o)
#pragma unroll
      for (int w = 0; w < TW; ++w) acc[o][w][0] = acc[o][w][1] = 0.0;

    for (int kc = 0; kc < kc_per; ++kc, ++g) {
      if (group == 0 && lt == 0 && kc == half && lw == 0 && lane == 0) mbar_arrive(go);
      const int s = g % Cfg::STAGES;
      mbar_wait(&full[s], (g / Cfg::STAGES) & 1);
      const double2* a2 = reinterpret_cast<const double2*>(sA + s * Cfg::A_STAGE);
      const double2* b2 = reinterpret_cast<const double2*>(sB + s * Cfg::B_STAGE);
#pragma unroll
      for (int ko = 0; ko < KO; ++ko) {
        double2 bf[TW], af[WO];
#pragma unroll
        for (int w = 0; w < TW; ++w) bf[w] = b2[(ko * (Cfg::BT / 8) + wt * TW + w) * 32 + lane];
#pragma unroll
        for (int o = 0; o < WO; ++o) af[o] = a2[(ko * (Cfg::BM / 8) + wm * WO + o) * 32 + lane];
#pragma unroll
        for (int o = 0; o < WO; ++o)
#pragma unroll
          for (int w = 0; w < TW; ++w) dmma(acc[o][w], af[o].x, bf[w].x);
#pragma unroll
        for (int o = 0; o < WO; ++o)
#pragma unroll
          for (int w = 0; w < TW; ++w) dmma(acc[o][w], af[o].y, bf[w].y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    if (args.rowmajor) {
      // out[i][j]: each lane holds a trait pair -> one 16-byte store
#pragma unroll
      for (int w = 0; w < TW; ++w) {
        const int j = tt * Cfg::BT + (wt * TW + w) * 8 + 2 * (lane & 3);
#pragma unroll
        for (int o = 0; o < WO; ++o) {
          const int64_t il = int64_t(tm) * Cfg::BM + (wm * WO + o) * 8 + (lane >> 2);
          if (il < args.rows)
            *reinterpret_cast<double2*>(out + il * args.ld + j) =
                make_double2(acc[o][w][0], acc[o][w][1]);
        }
      }
      continue;
    }
    // store S_BR[j][i]: lanes cover 8 SNPs x 4 trait pairs per accumulator block
#pragma unroll
    for (int w = 0; w < TW; ++w) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = tt * Cfg::BT + (wt * TW + w) * 8 + 2 * (lane & 3) + e;
        if (j >= args.t) continue;
        double* col = out + int64_t(j) * args.ld;
#pragma unroll
        for (int o = 0; o < WO; ++o) {
          const int64_t il = int64_t(tm) * Cfg::BM + (wm * WO + o) * 8 + (lane >> 2);
          if (il < args.rows) col[il] = acc[o][w][e];
        }
      }
    }
  }
}

// dst[i] = sum_{s < ksplit} part[s * stride + i], s in order (split-K GEMMs).
static __global__ void sum_partials_kernel(const double* __restrict__ part, int64_t stride, int ksplit,
                                    int64_t count, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    double v = part[i];
    for (int s = 1; s < ksplit; ++s) v += part[s * stride + i];
    dst[i] = v;
  }
}

template <class Cfg>
cudaError_t launch_sbr(const CUtensorMap& map_sq, const SbrArgs& a, int ctas, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(gls_sbr_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(Cfg::SMEM_BYTES));
  if (e != cudaSuccess) return e;
  gls_sbr_kernel<Cfg><<<ctas, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(map_sq, a);
  return cudaGetLastError();
}

// Instantiated S_BR configurations (kernels_lin_a.cu): tile shape + launcher.
struct SbrOps {
  int bm = 0, bt = 0, bk = 0;
  cudaError_t (*launch)(const CUtensorMap&, const SbrArgs&, int, cudaStream_t) = nullptr;
};
template <class Cfg>
SbrOps make_sbr_ops() {
  SbrOps o;
  o.bm = Cfg::BM;
  o.bt = Cfg::BT;
  o.bk = Cfg::BK;
  o.launch = &launch_sbr<Cfg>;
  return o;
}
// variant 0 = SbrDefault (64 SNPs x 64 traits); 1 = 128 x 40; 2 = 64 x 40
constexpr int kSbrConfigs = 3;
SbrOps sbr_ops(int variant);

}  // namespace gwg
