// kernel_table.cuh — per-p kernel instantiation table shared by the
// kernels_*.cu translation units (split so nvcc compiles them in parallel).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "grid_kernel.cuh"
#include "trait_prep.cuh"

namespace gwg {

#ifndef GWG_PRODUCER_WARP
#define GWG_PRODUCER_WARP true
#endif

constexpr int kBK = 32;  // k per pipeline stage; n is padded to a multiple of it

// ---------------------------------------------------------------------------
// Per-p kernel table.  Tile shapes keep p+1 accumulators per cell in
// registers and 3 smem stages under 227 KB:
//   p <= 6 : 64 SNPs x 32 traits per CTA, warp tile 32 x 8
//   p <= 12: 64 x 16, warp tile 16 x 8
//   p <= 32: 64 x 8,  warp tile 8 x 8
// ---------------------------------------------------------------------------
struct KernelOps {
  int bm = 0, bt = 0, bk = 0, groups = 1, threads = 0;
  size_t smem = 0;
  int ctx_stride = 0;
  cudaError_t (*prep)(const PrepArgs&, cudaStream_t) = nullptr;
  cudaError_t (*grid)(const CUtensorMap&, const CUtensorMap&, const GridArgs&, int,
                      cudaStream_t) = nullptr;
  // the same tiling with S_BR read from HBM (GridCfg::EXT; same panels)
  cudaError_t (*grid_ext)(const CUtensorMap&, const CUtensorMap&, const GridArgs&, int,
                          cudaStream_t) = nullptr;
};

template <class Cfg>
cudaError_t launch_grid(const CUtensorMap& map, const CUtensorMap& map_sq, const GridArgs& a,
                        int ctas, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(gls_grid_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(Cfg::SMEM_BYTES));
  if (e != cudaSuccess) return e;
  gls_grid_kernel<Cfg><<<ctas, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(map, map_sq, a);
  return cudaGetLastError();
}

#ifndef GWG_PINGPONG
#define GWG_PINGPONG 1
#endif

#ifndef GWG_PINGPONG_MAXP
#define GWG_PINGPONG_MAXP 12
#endif

template <int P, bool EXT = false>
struct CfgFor {
  static constexpr int LIM = 227 * 1024 - 128;
  // Ping-pong (two 4-warp consumer groups, one producer warp each), p <= 12:
  //   p <= 6 : group tile 64 SNPs x 16 traits, warp tile 32 x 8
  //   p <= 12: group tile 64 x 8, warp tile 16 x 8
  // p > 12: one group of 8 warps, tile 64 x 8, warp tile 8 x 8 (measured on
  // the B200: ping-pong with 32 x 8 group tiles is slower there, 31.1 vs
  // 32.2 TFLOP/s at p = 20; faster at p = 8 and 12, 31.6 vs 30.7 / 30.8 vs 29.8).
  static constexpr bool PP = GWG_PINGPONG && GWG_PRODUCER_WARP && P <= GWG_PINGPONG_MAXP;
  static constexpr int GROUPS = PP ? 2 : 1;
  static constexpr int WM_OCT = P <= 6 ? 4 : (P <= 12 ? 2 : 1);
  static constexpr int WARPS_T =
      PP ? (P <= 6 ? 2 : 1) : (P <= 6 ? 4 : (P <= 12 ? 2 : 1));
  static constexpr int WARPS_M = 8 / GROUPS / WARPS_T;
  static constexpr int BM = 8 * WM_OCT * WARPS_M;
  static constexpr int BT = 8 * WARPS_T;
  static constexpr int stage_bytes(int bk, bool ext) {
    return GROUPS * bk * ((ext ? 1 : 2) * BM + (ext ? P : P + 1) * BT) * 8;
  }
  static constexpr int MIN_ST = PP ? 2 : 3;
  // BK = 32 when MIN_ST stages of the fused kernel fit, else 16, with as
  // many stages as fit (<= 6); the EXT kernel keeps the fused kernel's BK
  // (measured: letting its smaller stages pick BK = 32 with 2 stages made
  // p = 12 78.7 ms instead of 46) and takes the extra stages instead
  static constexpr int BK = MIN_ST * stage_bytes(32, false) <= LIM ? 32 : 16;
  static constexpr int FIT = LIM / stage_bytes(BK, EXT);
  static constexpr int STAGES = FIT > 6 ? 6 : FIT;
  using type =
      GridCfg<P, WM_OCT, WARPS_M, WARPS_T, BK, STAGES, GWG_PRODUCER_WARP, GROUPS, EXT>;
};

template <int P>
KernelOps make_ops() {
  using Cfg = typename CfgFor<P>::type;
  static_assert(Cfg::SMEM_BYTES <= 227 * 1024, "shared memory budget");
  KernelOps k;
  k.bm = Cfg::BM;
  k.bt = Cfg::BT;
  k.bk = Cfg::BK;
  k.groups = Cfg::GROUPS;
  k.threads = Cfg::THREADS;
  k.smem = Cfg::SMEM_BYTES;
  k.ctx_stride = CtxLayout<P>::STRIDE;
  k.prep = &launch_trait_prep<P, Cfg::BT>;
  k.grid = &launch_grid<Cfg>;
  using Ext = typename CfgFor<P, true>::type;
  static_assert(Ext::BM == Cfg::BM && Ext::BT == Cfg::BT, "same tiles and panels");
  k.grid_ext = &launch_grid<Ext>;
  return k;
}

// One per translation unit (kernels_a.cu .. kernels_d.cu), compiled in parallel.
bool ops_for_a(int64_t p, KernelOps* out);
bool ops_for_b(int64_t p, KernelOps* out);
bool ops_for_c(int64_t p, KernelOps* out);
bool ops_for_d(int64_t p, KernelOps* out);

inline bool ops_for(int64_t p, KernelOps* out) {
  return ops_for_a(p, out) || ops_for_b(p, out) || ops_for_c(p, out) || ops_for_d(p, out);
}

}  // namespace gwg
