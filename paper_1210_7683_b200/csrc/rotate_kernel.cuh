// rotate_kernel.cuh — deterministic eigenbasis rotation dst = Z^T src (FP64 DMMA).
//
// Replaces rotate_columns / transform_snp_slab / transform_trait_slab
// (proj/src/grid.cpp:103-144).  The reference stages single columns through a
// two-column product so that every rotated column is bitwise independent of
// how columns are grouped into calls (grid.cpp:111-121); a library DGEMM picks
// different algorithms (tile shapes, split-K) for different widths and breaks
// that property.  This kernel fixes the reduction order of every output
// element — k-octets ascending, even k then odd k inside an octet, the DMMA's
// own order inside each — so X'[:, i] depends only on (Z, X[:, i]): results
// are bitwise identical for any slab width, slab offset or GPU count, and
// the grid results inherit that.
//
// GEMM view: M = eigen index r (n), N = columns i, K = samples k (n).  Both
// operands are K-contiguous in HBM (Z column r, src column i), so both are
// loaded by TMA 2-D boxes of (8 k x rows) into [k-octet][row][k%8] shared
// layout and read with conflict-free LDS.128 (each lane's two k values are
// adjacent).  CTA tile 128 r x 64 i, 8 warps of 32 r x 32 i plus a TMA
// producer warp, persistent static schedule.  For SNP slabs the
// epilogue also writes X'.X' (the A operand of S_BR = (X'.X')^T D), so the
// grid kernel never squares on the FP64 pipe that its DMMAs need.
#pragma once

#include <algorithm>

#include "gwg_device.cuh"

namespace gwg {

struct RotCfg {
  static constexpr int BM = 128;        // r per CTA
  static constexpr int BN = 64;         // columns per CTA
  static constexpr int WARPS_M = 4;     // warps along r (32 r each)
  static constexpr int WARPS_N = 2;     // warps along columns (32 each)
  static constexpr int WM_OCT = 4;      // r octets per warp
  static constexpr int WN_OCT = 4;      // column octets per warp
  static constexpr int BK = 32;
  static constexpr int STAGES = 4;
  static constexpr int WARPS = WARPS_M * WARPS_N;
  static constexpr int THREADS = (WARPS + 1) * 32;  // + one TMA producer warp
  static constexpr int A_STAGE = BK * BM;
  static constexpr int B_STAGE = BK * BN;
  static constexpr uint32_t STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
};

struct RotArgs {
  double* dst;        // n x cols, leading dimension ldd
  double* dst_sq;     // optional: elementwise squares of dst (same layout), or null
  int64_t ldd;
  int32_t n;          // rows of dst (= samples)
  int32_t cols;
  int32_t tiles_m;    // ceil(n / BM)
  int32_t tiles_n;    // ceil(cols / BN)
  int32_t kchunks;    // ceil(n / BK)
  const unsigned long long* gate = nullptr;  // GWG_SNP_AUTO path gate (gate_closed)
  int32_t gate_codes = 0;
};

__device__ __forceinline__ void rot_issue(const CUtensorMap* tz, const CUtensorMap* tx,
                                          const RotArgs& a, double* sA, double* sB,
                                          uint64_t* full, uint64_t* empty, int g, int total,
                                          uint64_t pol_z, uint64_t pol_x) {
  using C = RotCfg;
  if (g >= total) return;
  constexpr int KO = C::BK / 8;
  const int s = g % C::STAGES;
  const int use = g / C::STAGES;
  if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
  const int lt = g / a.kchunks;
  const int kc = g - lt * a.kchunks;
  const int tile = blockIdx.x + lt * gridDim.x;
  const int tn = tile / a.tiles_m;
  const int tm = tile - tn * a.tiles_m;
  mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
#pragma unroll
  for (int ko = 0; ko < KO; ++ko) {
    tma_load_2d(sA + s * C::A_STAGE + ko * C::BM * 8, tz, (kc * KO + ko) * 8, tm * C::BM,
                &full[s], pol_z);
    tma_load_2d(sB + s * C::B_STAGE + ko * C::BN * 8, tx, (kc * KO + ko) * 8, tn * C::BN,
                &full[s], pol_x);
  }
}

__global__ void __launch_bounds__(RotCfg::THREADS, 1)
    rotate_kernel(const __grid_constant__ CUtensorMap tmap_z,
                  const __grid_constant__ CUtensorMap tmap_x, const RotArgs a) {
  if (gate_closed(a.gate, a.gate_codes)) return;
  using C = RotCfg;
  constexpr int KO = C::BK / 8;
  extern __shared__ __align__(1024) double smem[];
  double* sA = smem;
  double* sB = sA + C::STAGES * C::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_STAGE);
  uint64_t* empty = full + C::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_n;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int total = my_tiles * a.kchunks;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == C::WARPS) {  // producer warp: one lane drives the TMA ring
    if (lane == 0) {
      const uint64_t pol_z = policy_evict_last();   // Z: shared by every CTA
      const uint64_t pol_x = policy_evict_first();  // source columns: read by tiles_m CTAs
      for (int g = 0; g < total; ++g)
        rot_issue(&tmap_z, &tmap_x, a, sA, sB, full, empty, g, total, pol_z, pol_x);
    }
    return;
  }
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  int g = 0;
  for (int lt = 0; lt < my_tiles; ++lt) {
    const int tile = blockIdx.x + lt * gridDim.x;
    const int tn = tile / a.tiles_m;
    const int tm = tile - tn * a.tiles_m;
    double acc[C::WM_OCT][C::WN_OCT][2];
#pragma unroll
    for (int i = 0; i < C::WM_OCT; ++i)
#pragma unroll
      for (int j = 0; j < C::WN_OCT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kc = 0; kc < a.kchunks; ++kc, ++g) {
      const int s = g % C::STAGES;
      mbar_wait(&full[s], (g / C::STAGES) & 1);
      const double2* a2 = reinterpret_cast<const double2*>(sA + s * C::A_STAGE);
      const double2* b2 = reinterpret_cast<const double2*>(sB + s * C::B_STAGE);
#pragma unroll
      for (int ko = 0; ko < KO; ++ko) {
        double2 af[C::WM_OCT], bf[C::WN_OCT];
#pragma unroll
        for (int i = 0; i < C::WM_OCT; ++i)
          af[i] = a2[(ko * (C::BM / 8) + wm * C::WM_OCT + i) * 32 + lane];
#pragma unroll
        for (int j = 0; j < C::WN_OCT; ++j)
          bf[j] = b2[(ko * (C::BN / 8) + wn * C::WN_OCT + j) * 32 + lane];
#pragma unroll
        for (int i = 0; i < C::WM_OCT; ++i)
#pragma unroll
          for (int j = 0; j < C::WN_OCT; ++j) dmma(acc[i][j], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < C::WM_OCT; ++i)
#pragma unroll
          for (int j = 0; j < C::WN_OCT; ++j) dmma(acc[i][j], af[i].y, bf[j].y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // store: acc[i][j][e] = dst[r][col], r = row octet i, col = 2(lane&3)+e of octet j
    const uint64_t pol_out = policy_evict_first();
#pragma unroll
    for (int i = 0; i < C::WM_OCT; ++i) {
      const int r = tm * C::BM + (wm * C::WM_OCT + i) * 8 + (lane >> 2);
      if (r >= a.n) continue;
#pragma unroll
      for (int j = 0; j < C::WN_OCT; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = tn * C::BN + (wn * C::WN_OCT + j) * 8 + 2 * (lane & 3) + e;
          if (col < a.cols) {
            st_evict_first(a.dst + int64_t(col) * a.ldd + r, acc[i][j][e], pol_out);
            if (a.dst_sq)
              st_evict_first(a.dst_sq + int64_t(col) * a.ldd + r, acc[i][j][e] * acc[i][j][e],
                             pol_out);
          }
        }
      }
    }
  }
}

}  // namespace gwg

namespace gwg {

inline cudaError_t launch_rotate(const CUtensorMap& tz, const CUtensorMap& tx, const RotArgs& a,
                                 int ctas, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(RotCfg::SMEM_BYTES));
  if (e != cudaSuccess) return e;
  rotate_kernel<<<ctas, RotCfg::THREADS, RotCfg::SMEM_BYTES, s>>>(tz, tx, a);
  return cudaGetLastError();
}

// Elementwise squares for slabs that arrive already rotated.
__global__ void square_kernel(const double* __restrict__ x, double* __restrict__ y, size_t count) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x)
    y[i] = x[i] * x[i];
}

inline cudaError_t launch_square(const double* x, double* y, size_t count, cudaStream_t s) {
  const int blocks = int(std::min<size_t>((count + 255) / 256, 148 * 16));
  square_kernel<<<blocks, 256, 0, s>>>(x, y, count);
  return cudaGetLastError();
}

}  // namespace gwg
