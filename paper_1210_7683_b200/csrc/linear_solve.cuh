// linear_solve.cuh — second launch of the genotype split grid (grid_split.cuh):
// the p linear terms of every cell exactly on the int8 tensor cores, and the
// cell's bordered Cholesky solve in the same epilogue.
//
// GEMM view per CTA tile: M = 128 SNPs (A = int8 genotype codes, K-major),
// N = 8 slices x RB rows of W (B, K-major), K = samples; int32 accumulators in
// TMEM, double-buffered (the TMA producer / MMA issuer / TMEM code is shared
// with rotate_i8_kernel).  W is laid out per tile of KT traits, each trait's p
// columns padded to P8 (a power of two <= 8, else a multiple of 8) so that a
// trait's columns are one aligned tcgen05.ld.
//
// Epilogue (8 warps, two per TMEM lane quarter; thread = SNP row): per cell
// (i, j) the p linear terms x_i^T W_{j,c} are recombined exactly from the
// eight slice products (i8_recombine, one rounding), S_BR[j][i] comes from
// gls_sbr_kernel (prefetched before the accumulator wait), and solve_cell<P>
// — the same bordered Cholesky as the all-FP64 kernel — produces b_ij, which
// leaves through a 128B-swizzled staging tile and a TMA store (numpy layout)
// or direct stores (stream layout).  Failed cells: NaN + the min error key,
// exactly like gls_grid_kernel.
#pragma once

#include "grid_kernel.cuh"
#include "i8_core.cuh"

namespace gwg {

template <int P>
struct LinCfg {
  static constexpr int P8 = P <= 1 ? 1 : P <= 2 ? 2 : P <= 4 ? 4 : P <= 8 ? 8 : (P + 7) / 8 * 8;
  static constexpr int KT = 32 / P8 >= 1 ? 32 / P8 : 1;  // traits per tile
  static constexpr int RB = KT * P8;                      // W rows per tile (24 or 32)
  using Tile = I8Tile<RB>;
  static constexpr int HALVES = KT >= 2 ? 2 : 1;          // epilogue warps per lane quarter in use
  static constexpr int CELLS = KT >= 2 ? KT / 2 : 1;      // cells per epilogue thread per tile
  static constexpr int CW = P8 < 8 ? P8 : 8;              // TMEM columns per load
  static constexpr bool TMA_OUT = CELLS * P == Tile::OUT_Q;  // a 128-byte row per thread
};

struct LinArgs {
  const double* scale;  // sigma per (padded) W row
  const double* sbr;    // S_BR[j * ld_s + i] from gls_sbr_kernel
  int64_t ld_s;
  const double* ctx;    // per-trait contexts (CtxLayout<P>)
  double* out;
  int64_t out_si;       // cell strides of out
  int64_t out_sj;
  int32_t use_tma;      // out through tmap_out (numpy layout, 16-byte pitch)
  int32_t t;
  int64_t rows;
  int64_t i0;
  int64_t m_total;
  int32_t tiles_m;
  int32_t tiles_r;      // ceil(t / KT)
  int32_t kstages;
  unsigned long long* err_key;
};

template <int P>
__global__ void __launch_bounds__(LinCfg<P>::Tile::THREADS, 1)
    linear_solve_kernel(const __grid_constant__ CUtensorMap tmap_x,
                        const __grid_constant__ CUtensorMap tmap_w,
                        const __grid_constant__ CUtensorMap tmap_out, const LinArgs a) {
  using L = LinCfg<P>;
  using C = typename L::Tile;
  using CX = CtxLayout<P>;
  constexpr int CELLS = L::CELLS;
  extern __shared__ __align__(1024) unsigned char smem_ls[];
  const I8Smem<C> sm(smem_ls);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_r;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t tmem_base = i8_setup<C>(sm, warp);

  if (warp == 0) {
    if (lane == 0) i8_produce<C>(sm, &tmap_x, &tmap_w, my_tiles, a.tiles_r, a.kstages);
  } else if (warp == 1) {
    if (lane == 0) i8_mma<C>(sm, tmem_base, my_tiles, a.kstages);
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int qd = warp & 3;
    const int h = ew >> 2;
    const bool active = h < L::HALVES;
    unsigned char* stg = sm.staging + ew * C::OUT_BYTES;
    for (int lt = 0; lt < my_tiles; ++lt) {
      const int buf = lt & 1;
      const int tile = blockIdx.x + lt * gridDim.x;
      const int tm = tile / a.tiles_r;
      const int tr = tile - tm * a.tiles_r;
      const int64_t il = int64_t(tm) * C::BM + qd * 32 + lane;
      const bool iv = il < a.rows;
      const int j0 = tr * L::KT + h * CELLS;  // first trait of this warp
      double sbr[CELLS];
#pragma unroll
      for (int cc = 0; cc < CELLS; ++cc) {
        const int j = j0 + cc;
        sbr[cc] = (active && iv && j < a.t) ? __ldcs(a.sbr + int64_t(j) * a.ld_s + il) : 0.0;
      }
      mbar_wait(&sm.acc_full[buf], (lt >> 1) & 1);
      tc_fence_after();
      double lin[CELLS][P];
      if (active) {
        const uint32_t taddr = tmem_base + (uint32_t(qd * 32) << 16) + uint32_t(buf * C::BN);
#pragma unroll
        for (int cc = 0; cc < CELLS; ++cc) {
          const int col0 = (h * CELLS + cc) * L::P8;
#pragma unroll
          for (int c0 = 0; c0 < P; c0 += L::CW) {
            int32_t v[C::SLICES][L::CW];
#pragma unroll
            for (int sl = 0; sl < C::SLICES; ++sl)
              tmem_ldw<L::CW>(taddr + uint32_t(sl * C::RB + col0 + c0), v[sl]);
            tmem_ld_wait();
#pragma unroll
            for (int r = 0; r < L::CW; ++r) {
              if (c0 + r < P) {
                const double sc = __ldg(a.scale + tr * C::RB + col0 + c0 + r);
                lin[cc][c0 + r] = i8_recombine(v[0][r], v[1][r], v[2][r], v[3][r], v[4][r],
                                               v[5][r], v[6][r], v[7][r], sc);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.acc_empty[buf]);  // TMEM buffer free for the next tile
      if (!active) continue;

      // ---- bordered Cholesky per cell (FP64 pipe; no DMMA in this kernel) ----
      double beta[CELLS][P];
#pragma unroll
      for (int cc = 0; cc < CELLS; ++cc) {
        const int j = j0 + cc;
        if (j < a.t && iv) {
          double cell[P + 1];
#pragma unroll
          for (int c = 0; c < P; ++c) cell[c] = lin[cc][c];
          cell[P] = sbr[cc];
          const bool ok = solve_cell<P>(cell, a.ctx + size_t(j) * CX::STRIDE, beta[cc]);
          if (!ok) {
            atomicMin(a.err_key, (unsigned long long)(int64_t(j) * a.m_total + a.i0 + il));
#pragma unroll
            for (int c = 0; c < P; ++c) beta[cc][c] = __longlong_as_double(0x7ff8000000000000LL);
          }
        } else {
#pragma unroll
          for (int c = 0; c < P; ++c) beta[cc][c] = 0.0;
        }
      }
      bool stored = false;
      if constexpr (L::TMA_OUT) {
        if (a.use_tma) {
          stored = true;
          if (lane == 0) bulk_wait_read0();  // the previous store has left the staging tile
          __syncwarp();
#pragma unroll
          for (int ch = 0; ch < C::OUT_Q / 2; ++ch) {
            const int f = 2 * ch;
            double2 w;
            w.x = beta[f / P][f % P];
            w.y = beta[(f + 1) / P][(f + 1) % P];
            *reinterpret_cast<double2*>(stg + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tma_store_2d(&tmap_out, stg, j0 * P, tm * C::BM + qd * 32);
        }
      }
      if (!stored && iv) {
#pragma unroll
        for (int cc = 0; cc < CELLS; ++cc) {
          const int j = j0 + cc;
          if (j >= a.t) continue;
          double* dst = a.out + (il * a.out_si + int64_t(j) * a.out_sj) * P;
#pragma unroll
          for (int c = 0; c < P; ++c) __stcs(dst + c, beta[cc][c]);
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  i8_teardown<C>(tmem_base, warp);
}

template <int P>
cudaError_t launch_linear_solve(const CUtensorMap& tx, const CUtensorMap& tw,
                                const CUtensorMap& tout, const LinArgs& a, int ctas,
                                cudaStream_t s) {
  using C = typename LinCfg<P>::Tile;
  cudaError_t e = cudaFuncSetAttribute(linear_solve_kernel<P>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(C::SMEM_BYTES));
  if (e != cudaSuccess) return e;
  linear_solve_kernel<P><<<ctas, C::THREADS, C::SMEM_BYTES, s>>>(tx, tw, tout, a);
  return cudaGetLastError();
}

// Per-p entry of the split grid (kernels_lin_*.cu).
struct LinOps {
  int kt = 0, p8 = 0, rb = 0;
  cudaError_t (*launch)(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                        const LinArgs&, int, cudaStream_t) = nullptr;
};

template <int P>
LinOps make_lin_ops() {
  LinOps o;
  o.kt = LinCfg<P>::KT;
  o.p8 = LinCfg<P>::P8;
  o.rb = LinCfg<P>::RB;
  o.launch = &launch_linear_solve<P>;
  return o;
}

bool lin_ops_for_a(int64_t p, LinOps* out);  // p 1..16
bool lin_ops_for_b(int64_t p, LinOps* out);  // p 17..32
inline bool lin_ops_for(int64_t p, LinOps* out) {
  return lin_ops_for_a(p, out) || lin_ops_for_b(p, out);
}

}  // namespace gwg
