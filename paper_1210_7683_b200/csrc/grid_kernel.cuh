// grid_kernel.cuh — the fused GLS-grid kernel (sm_100a, FP64 DMMA).
//
// Replaces compute_tile -> compute_block -> solve_gls_cell
// (proj/src/grid.cpp:191-273, proj/src/gls.cpp:105-132).  For every cell
// (SNP i, trait j) the reference forms w_r = k.x'_i and reduces it against the
// trait context (S_BL = w_r^T w_l, S_BR = |w_r|^2, b_B = w_r.v), then LLT-solves
// the p x p system.  With D_j = 1/d_j = k_j^2 those reductions are three dense
// contractions over n:
//     S_BL[i,j,l] = X'^T (D.X_L'_l)     b_B[i,j] = X'^T (D.Y')
//     S_BR[i,j]   = (X'.X')^T D
// i.e. one GEMM with M = SNPs, N = traits x (p+1) operand columns, K = n, run
// on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4).  X'.X' is formed
// by squaring the A fragment in registers.  The p+1 accumulators of a cell
// land in the same thread (the N axis is ordered component-major inside each
// 8-trait octet), so the bordered Cholesky solve against the per-trait
// chol(S_TL) and the store of b_ij happen in registers: no m x t intermediate
// ever reaches HBM.
//
// Data path (per CTA, persistent over tiles):
//   producer warp : TMA 2-D loads of the rotated SNP tile (box 8 k x BM SNPs,
//                   one per k-octet; zero-filled past n and past m) and one
//                   1-D bulk copy of the pre-laid-out trait-operand stage,
//                   STAGES-deep mbarrier ring.
//   consumer warps: WARPS_M x WARPS_T warps, warp tile (8*WM_OCT SNPs) x
//                   (8 traits) x (p+1) operand columns; LDS.128 fragment
//                   loads (each lane's pair of k values is contiguous, so a
//                   warp load is 512 contiguous bytes: no bank conflicts).
//
// Shared-memory stage layouts (doubles):
//   A[kc][i][kk]            kc < BK/8, i < BM, kk < 8         (TMA box order)
//   B[kc][c][g][jj][kk]     c < p+1, g < BT/8, jj < 8, kk < 8 (panel order)
// The contraction order over k is fixed (k-octets ascending; within an octet
// the even k then the odd k; DMMA-internal order within each) and independent
// of how SNPs/traits are tiled, sharded or slabbed, so b is bitwise identical
// across slab widths and GPU counts.
#pragma once

#include "gwg_device.cuh"

namespace gwg {

// Per-trait epilogue context: 1/L_aa (p-1), strictly-lower L (packed by rows),
// z = L^-1 b_T (p-1), flag (0 ok, else chol(S_TL) failed).
template <int P>
struct CtxLayout {
  static constexpr int P1 = P - 1;
  static constexpr int NOFF = P1 > 1 ? P1 * (P1 - 1) / 2 : 0;
  static constexpr int INVD = 0;
  static constexpr int OFF = P1;
  static constexpr int Z = P1 + NOFF;
  static constexpr int FLAG = 2 * P1 + NOFF;
  static constexpr int STRIDE = (FLAG + 2) & ~1;
  __host__ __device__ static constexpr int off_idx(int a, int c) { return a * (a - 1) / 2 + c; }
};

template <int P_, int WM_OCT_, int WARPS_M_, int WARPS_T_, int BK_, int STAGES_>
struct GridCfg {
  static constexpr int P = P_;
  static constexpr int NC = P + 1;  // operand columns per trait
  static constexpr int WM_OCT = WM_OCT_;
  static constexpr int WARPS_M = WARPS_M_;
  static constexpr int WARPS_T = WARPS_T_;
  static constexpr int BK = BK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int BM = 8 * WM_OCT * WARPS_M;
  static constexpr int BT = 8 * WARPS_T;
  static constexpr int CONSUMER_WARPS = WARPS_M * WARPS_T;
  static constexpr int THREADS = (CONSUMER_WARPS + 1) * 32;
  static constexpr int A_STAGE = BK * BM;        // doubles
  static constexpr int B_STAGE = BK * NC * BT;   // doubles
  static constexpr uint32_t A_BYTES = A_STAGE * 8;
  static constexpr uint32_t B_BYTES = B_STAGE * 8;
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * (A_BYTES + B_BYTES) + 2 * STAGES * sizeof(uint64_t) + 1024;
  static_assert(BK % 8 == 0, "BK must be a multiple of 8");
  static_assert(BM <= 256, "TMA box outer dimension is at most 256");
};

struct GridArgs {
  const double* bops;   // trait-operand panels (see trait_prep)
  const double* ctx;    // per-trait epilogue contexts
  double* out;          // results
  int64_t out_si;       // cell stride (in cells) per local SNP row
  int64_t out_sj;       // cell stride (in cells) per trait
  int64_t rows;         // valid SNP rows in this slab
  int64_t i0;           // global index of slab row 0
  int64_t m_total;      // global SNP count (error key)
  int32_t t;            // valid traits
  int32_t tiles_m;
  int32_t tiles_t;
  int32_t kchunks;      // NP / BK
  int64_t np;           // padded n (multiple of BK)
  unsigned long long* err_key;  // min over failing cells of j*m_total + i
};

// Bordered Cholesky solve of one cell.  The leading (p-1) block of chol(S) is
// chol(S_TL) (computed once per trait), so only the last row is per cell:
//   l = L^-1 s_bl,  pivot = s_br - |l|^2  (fails iff pivot <= 0, like Eigen's
//   LLT: NaN passes), lambda = sqrt(pivot), then forward/back substitution.
template <int P>
__device__ __forceinline__ bool solve_cell(const double* acc, const double* __restrict__ cx,
                                           double* beta) {
  using L = CtxLayout<P>;
  constexpr int P1 = L::P1;
  double l[P1 > 0 ? P1 : 1];
#pragma unroll
  for (int a = 0; a < P1; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < a; ++c) s = fma(__ldg(cx + L::OFF + L::off_idx(a, c)), l[c], s);
    l[a] = (acc[a] - s) * __ldg(cx + L::INVD + a);
  }
  double sq = 0.0, lz = 0.0;
#pragma unroll
  for (int a = 0; a < P1; ++a) {
    sq = fma(l[a], l[a], sq);
    lz = fma(l[a], __ldg(cx + L::Z + a), lz);
  }
  const double pivot = acc[P] - sq;
  const bool ok = !(pivot <= 0.0) && __ldg(cx + L::FLAG) == 0.0;
  const double lam = sqrt(pivot);
  const double bb = ((acc[P1] - lz) / lam) / lam;
  beta[P1] = bb;
#pragma unroll
  for (int a = P1 - 1; a >= 0; --a) {
    double r = __ldg(cx + L::Z + a) - l[a] * bb;
#pragma unroll
    for (int c = a + 1; c < P1; ++c) r -= __ldg(cx + L::OFF + L::off_idx(c, a)) * beta[c];
    beta[a] = r * __ldg(cx + L::INVD + a);
  }
  return ok;
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    gls_grid_kernel(const __grid_constant__ CUtensorMap tmap_a, const GridArgs args) {
  constexpr int P = Cfg::P;
  constexpr int NC = Cfg::NC;
  constexpr int P1 = P - 1;
  constexpr int KO = Cfg::BK / 8;  // k-octets per stage
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* sA = reinterpret_cast<double*>(base);
  double* sB = sA + Cfg::STAGES * Cfg::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + Cfg::STAGES * Cfg::B_STAGE);
  uint64_t* empty = full + Cfg::STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::CONSUMER_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int ntiles = args.tiles_m * args.tiles_t;

  if (warp == Cfg::CONSUMER_WARPS) {
    // ---------------- producer: one elected lane drives the TMA ring ----------
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();    // trait operands: L2-resident
      const uint64_t stream = policy_evict_first();  // SNP tiles: read ~once
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tm = tile / args.tiles_t;
        const int tt = tile - tm * args.tiles_t;
        const double* bsrc = args.bops + size_t(tt) * size_t(args.np) * NC * Cfg::BT;
        for (int kc = 0; kc < args.kchunks; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::A_BYTES + Cfg::B_BYTES);
          double* a_dst = sA + stage * Cfg::A_STAGE;
#pragma unroll
          for (int ko = 0; ko < KO; ++ko)
            tma_load_2d(a_dst + ko * Cfg::BM * 8, &tmap_a, (kc * KO + ko) * 8, tm * Cfg::BM,
                        &full[stage], stream);
          bulk_load(sB + stage * Cfg::B_STAGE, bsrc + size_t(kc) * Cfg::B_STAGE, Cfg::B_BYTES,
                    &full[stage], keep);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers -------------------------------------------------
  const int wm = warp % Cfg::WARPS_M;
  const int wt = warp / Cfg::WARPS_M;
  int stage = 0;
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tm = tile / args.tiles_t;
    const int tt = tile - tm * args.tiles_t;

    double acc[Cfg::WM_OCT][NC][2];
#pragma unroll
    for (int o = 0; o < Cfg::WM_OCT; ++o)
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[o][c][0] = acc[o][c][1] = 0.0;

    for (int kc = 0; kc < args.kchunks; ++kc) {
      mbar_wait(&full[stage], phase);
      const double2* a2 = reinterpret_cast<const double2*>(sA + stage * Cfg::A_STAGE);
      const double2* b2 = reinterpret_cast<const double2*>(sB + stage * Cfg::B_STAGE);
#pragma unroll
      for (int ko = 0; ko < KO; ++ko) {
        double2 bf[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c)
          bf[c] = b2[((ko * NC + c) * Cfg::WARPS_T + wt) * 32 + lane];
#pragma unroll
        for (int o = 0; o < Cfg::WM_OCT; ++o) {
          const double2 af = a2[(ko * (Cfg::BM / 8) + wm * Cfg::WM_OCT + o) * 32 + lane];
          const double sqx = af.x * af.x, sqy = af.y * af.y;
#pragma unroll
          for (int c = 0; c < P; ++c) {
            dmma(acc[o][c], af.x, bf[c].x);
            dmma(acc[o][c], af.y, bf[c].y);
          }
          dmma(acc[o][P], sqx, bf[P].x);
          dmma(acc[o][P], sqy, bf[P].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == Cfg::STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    // ---------------- fused epilogue: bordered Cholesky + store -----------------
    using L = CtxLayout<P>;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = tt * Cfg::BT + wt * 8 + 2 * (lane & 3) + e;
      if (j >= args.t) continue;
      const double* cx = args.ctx + size_t(j) * L::STRIDE;
#pragma unroll
      for (int o = 0; o < Cfg::WM_OCT; ++o) {
        const int64_t il = int64_t(tm) * Cfg::BM + (wm * Cfg::WM_OCT + o) * 8 + (lane >> 2);
        if (il >= args.rows) continue;
        double cell[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) cell[c] = acc[o][c][e];
        double beta[P];
        const bool ok = solve_cell<P>(cell, cx, beta);
        double* dst = args.out + (il * args.out_si + int64_t(j) * args.out_sj) * P;
        if (!ok) {
          atomicMin(args.err_key,
                    (unsigned long long)(int64_t(j) * args.m_total + args.i0 + il));
#pragma unroll
          for (int c = 0; c < P; ++c) beta[c] = __longlong_as_double(0x7ff8000000000000LL);
        }
#pragma unroll
        for (int c = 0; c < P; ++c) __stcs(dst + c, beta[c]);
      }
    }
    (void)P1;
  }
}

}  // namespace gwg
