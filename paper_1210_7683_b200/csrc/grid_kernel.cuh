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
// on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4).  X'.X' comes
// precomputed from the rotation epilogue (squaring here would repeat the DMULs
// once per trait tile and steal FP64-pipe cycles from the DMMAs).  The p+1
// accumulators of a cell
// land in the same thread (the N axis is ordered component-major inside each
// 8-trait octet), so the bordered Cholesky solve against the per-trait
// chol(S_TL) and the store of b_ij happen in registers: no m x t intermediate
// ever reaches HBM.
//
// Data path (per CTA, persistent over tiles, 8 warps = 2 per SM sub-partition
// so each thread may hold up to 255 registers):
//   producer      : thread 0, inside the k loop, issues TMA 2-D loads of the
//                   rotated SNP tile (box 8 k x BM SNPs, one per k-octet;
//                   zero-filled past n and past m) and one 1-D bulk copy of the
//                   pre-laid-out trait-operand stage, STAGES-deep mbarrier ring
//                   with STAGES-2 stages in flight.
//   consumer warps: WARPS_M x WARPS_T warps, warp tile (8*WM_OCT SNPs) x
//                   (8 traits) x (p+1) operand columns; LDS.128 fragment
//                   loads (each lane's pair of k values is contiguous, so a
//                   warp load is 512 contiguous bytes: no bank conflicts).
//
// Shared-memory stage layouts (doubles):
//   A[kc][i][kk], then the same for X'.X'   kc < BK/8, i < BM, kk < 8 (TMA box)
//   B[kc][c][g][jj][kk]     c < p+1, g < BT/8, jj < 8, kk < 8 (panel order)
// The contraction order over k is fixed (k-octets ascending; within an octet
// the even k then the odd k; DMMA-internal order within each) and independent
// of how SNPs/traits are tiled, sharded or slabbed, so b is bitwise identical
// across slab widths and GPU counts.
#pragma once

#include "gwg_device.cuh"

// Timing experiments only (never in a shipped build): 1 = skip the Cholesky
// epilogue math, 2 = feed every k-chunk from the first STAGES loads.
#ifndef GWG_EXPERIMENT
#define GWG_EXPERIMENT 0
#endif
#ifndef GWG_RCP_MAXP
#define GWG_RCP_MAXP 4
#endif

namespace gwg {

// Per-trait epilogue context: 1/L_aa (p-1), strictly-lower L (packed by rows),
// z = L^-1 b_T (p-1), flag (0 ok, else chol(S_TL) failed), the full lower
// triangle of L^-1 (packed by rows) for solve_cell_inv, and c_T = L^-T z
// (= S_TL^-1 b_T, p-1) for the genotype grid's folded solve.
template <int P>
struct CtxLayout {
  static constexpr int P1 = P - 1;
  static constexpr int NOFF = P1 > 1 ? P1 * (P1 - 1) / 2 : 0;
  static constexpr int INVD = 0;
  static constexpr int OFF = P1;
  static constexpr int Z = P1 + NOFF;
  static constexpr int FLAG = 2 * P1 + NOFF;
  static constexpr int LINV = FLAG + 1;
  static constexpr int NLINV = P1 * (P1 + 1) / 2;
  static constexpr int CT = LINV + NLINV;
  static constexpr int STRIDE = (CT + P1 + 1) & ~1;
  __host__ __device__ static constexpr int off_idx(int a, int c) { return a * (a - 1) / 2 + c; }
  __host__ __device__ static constexpr int linv_idx(int a, int c) { return a * (a + 1) / 2 + c; }
};

template <int P_, int WM_OCT_, int WARPS_M_, int WARPS_T_, int BK_, int STAGES_,
          bool PRODUCER_WARP_ = true, int GROUPS_ = 1, bool EXT_ = false>
struct GridCfg {
  static constexpr int P = P_;
  static constexpr int NC = P + 1;  // operand columns per trait in the panels (trait_prep)
  // EXT: S_BR comes from HBM (the factorised ((X'.X')^T E) F of grid_split.cuh)
  // instead of the D column against X'.X': the stages hold X' and the first P
  // panel columns only, and the cell's last accumulator is not computed.
  static constexpr bool EXT = EXT_;
  static constexpr int NCS = EXT ? P : P + 1;  // panel columns staged and multiplied
  static constexpr int WM_OCT = WM_OCT_;
  static constexpr int WARPS_M = WARPS_M_;  // per consumer group
  static constexpr int WARPS_T = WARPS_T_;  // per consumer group
  static constexpr int BK = BK_;
  static constexpr int STAGES = STAGES_;    // per consumer group
  // PRODUCER_WARP: one extra warp per consumer group drives that group's TMA
  // ring (STAGES in flight).  Otherwise thread 0 issues inside the k loop with
  // LOOKAHEAD stages in flight.  GROUPS = 2 is the ping-pong schedule: two
  // consumer groups (one warp of each per SM sub-partition) work on adjacent
  // trait tiles half a tile out of phase, so one group's epilogue overlaps the
  // other's DMMA main loop.
  static constexpr bool PRODUCER_WARP = PRODUCER_WARP_;
  static constexpr int GROUPS = GROUPS_;
  static constexpr int LOOKAHEAD = STAGES - 2;
  static constexpr int BM = 8 * WM_OCT * WARPS_M;
  static constexpr int BT = 8 * WARPS_T;     // traits per group tile
  static constexpr int GWARPS = WARPS_M * WARPS_T;
  static constexpr int WARPS = GWARPS * GROUPS;
  static constexpr int THREADS = (WARPS + (PRODUCER_WARP ? GROUPS : 0)) * 32;
  static constexpr int A_STAGE = BK * BM;        // doubles (X' tile; X'.X' tile follows)
  static constexpr int B_STAGE = BK * NCS * BT;  // doubles staged
  static constexpr int B_GSTAGE = BK * NC * BT;  // panel doubles per k-chunk in HBM
  static constexpr uint32_t A_BYTES = (EXT ? 1 : 2) * A_STAGE * 8;
  static constexpr uint32_t B_BYTES = B_STAGE * 8;
  static constexpr int SA_STAGE = (EXT ? 1 : 2) * A_STAGE;  // smem doubles per stage: A (, A.A)
  static constexpr size_t SMEM_BYTES =
      size_t(GROUPS) * (size_t(STAGES) * (A_BYTES + B_BYTES) + 2 * STAGES * sizeof(uint64_t)) +
      sizeof(uint64_t);
  static_assert(BK % 8 == 0, "BK must be a multiple of 8");
  static_assert(BM <= 256, "TMA box outer dimension is at most 256");
  static_assert(PRODUCER_WARP || STAGES >= 3, "the in-loop producer needs one slack stage");
  static_assert(PRODUCER_WARP || GROUPS == 1, "ping-pong needs producer warps");
  static_assert(WARPS == 8, "two consumer warps per SM sub-partition");
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
  const double* sbr = nullptr;  // EXT: S_BR[j * ld_s + i]
  int64_t ld_s = 0;
  const unsigned long long* gate = nullptr;  // GWG_SNP_AUTO path gate (gate_closed)
  int32_t gate_codes = 0;
};

// Bordered Cholesky solve of one cell.  The leading (p-1) block of chol(S) is
// chol(S_TL) (computed once per trait), so only the last row is per cell:
//   l = L^-1 s_bl            (Eigen LLT's last-row update, divisions by L_aa
//                             folded into the stored reciprocals)
//   pivot = s_br - |l|^2     fails iff pivot <= 0, like Eigen's LLT (NaN passes)
//   beta_B = (b_B - l.z_T) / pivot     (= ((b_B - l.z_T)/lambda)/lambda;
//                                       reciprocal by rcp.approx + Newton)
//   beta_T = L^-T (z_T - l beta_B)
// 1/x by the MUFU approximation and two Newton steps (<= 1 ulp for normal
// x; far cheaper on the FP64 pipe than an IEEE division).  Flushes subnormal
// x to zero (callers divide exactly in that case).
__device__ __forceinline__ double rcp_newton(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}

// Context loads: read-only global (__ldg) or, SMEM, a shared-memory copy.
template <bool SMEM>
__device__ __forceinline__ double ctx_ld(const double* p) {
  if constexpr (SMEM)
    return *p;
  else
    return __ldg(p);
}

template <int P, bool SMEM = false>
__device__ __forceinline__ bool solve_cell(const double* acc, const double* __restrict__ cx,
                                           double* beta) {
  using L = CtxLayout<P>;
  constexpr int P1 = L::P1;
  double l[P1 > 0 ? P1 : 1];
#pragma unroll
  for (int a = 0; a < P1; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < a; ++c) s = fma(ctx_ld<SMEM>(cx + L::OFF + L::off_idx(a, c)), l[c], s);
    l[a] = (acc[a] - s) * ctx_ld<SMEM>(cx + L::INVD + a);
  }
  double sq = 0.0, lz = 0.0;
#pragma unroll
  for (int a = 0; a < P1; ++a) {
    sq = fma(l[a], l[a], sq);
    lz = fma(l[a], ctx_ld<SMEM>(cx + L::Z + a), lz);
  }
  const double pivot = acc[P] - sq;
  const bool ok = !(pivot <= 0.0) && ctx_ld<SMEM>(cx + L::FLAG) == 0.0;
  // 1/pivot: MUFU approximation + two Newton steps (<= 1 ulp; far cheaper on
  // the FP64 pipe than an IEEE division, which the other ping-pong group's
  // DMMAs are competing for)
  double bb;
  if (P <= GWG_RCP_MAXP) {
    double r;
    r = rcp_newton(pivot);
    bb = (acc[P1] - lz) * r;
    // a subnormal pivot is flushed by the approximation: divide exactly (the
    // reference's LLT accepts any positive pivot)
    if (pivot < 0x1p-1022 && pivot > 0.0) bb = (acc[P1] - lz) / pivot;
  } else {  // large p: the O(p^2) substitutions dominate; keep register pressure low
    bb = (acc[P1] - lz) / pivot;
  }
  beta[P1] = bb;
#pragma unroll
  for (int a = P1 - 1; a >= 0; --a) {
    double r = ctx_ld<SMEM>(cx + L::Z + a) - l[a] * bb;
#pragma unroll
    for (int c = a + 1; c < P1; ++c) r -= ctx_ld<SMEM>(cx + L::OFF + L::off_idx(c, a)) * beta[c];
    beta[a] = r * ctx_ld<SMEM>(cx + L::INVD + a);
  }
  return ok;
}

// The same bordered solve with the triangular solves done as products with
// the precomputed L^-1 (trait_prep), so the p-1 components of l and of beta_T
// are independent dot products instead of serial substitution chains: for
// large p the epilogue is latency-bound on those chains.  Same algebra,
// different rounding (well-conditioned S_TL); the pivot test is unchanged.
//   l = L^-1 s_bl,  pivot = s_br - |l|^2,  beta_B = (b_B - l.z_T) / pivot,
//   beta_T = L^-T (z_T - l beta_B)
template <int P, bool SMEM = false>
__device__ __forceinline__ bool solve_cell_inv(const double* acc, const double* __restrict__ cx,
                                               double* beta) {
  using L = CtxLayout<P>;
  constexpr int P1 = L::P1;
  double l[P1 > 0 ? P1 : 1];
#pragma unroll
  for (int a = 0; a < P1; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c <= a; ++c) s = fma(ctx_ld<SMEM>(cx + L::LINV + L::linv_idx(a, c)), acc[c], s);
    l[a] = s;
  }
  double sq = 0.0, lz = 0.0;
#pragma unroll
  for (int a = 0; a < P1; ++a) {
    sq = fma(l[a], l[a], sq);
    lz = fma(l[a], ctx_ld<SMEM>(cx + L::Z + a), lz);
  }
  const double pivot = acc[P] - sq;
  const bool ok = !(pivot <= 0.0) && ctx_ld<SMEM>(cx + L::FLAG) == 0.0;
  const double bb = (acc[P1] - lz) / pivot;
  beta[P1] = bb;
  double r[P1 > 0 ? P1 : 1];
#pragma unroll
  for (int a = 0; a < P1; ++a) r[a] = fma(-l[a], bb, ctx_ld<SMEM>(cx + L::Z + a));
#pragma unroll
  for (int c = 0; c < P1; ++c) {
    double s = 0.0;
#pragma unroll
    for (int a = c; a < P1; ++a) s = fma(ctx_ld<SMEM>(cx + L::LINV + L::linv_idx(a, c)), r[a], s);
    beta[c] = s;
  }
  return ok;
}

// The genotype grid's solve with L^-1 folded into W on the trait side
// (fold_w_kernel): the int8 MMA already yields l = L^-1 s_bl (acc[0..p-2])
// and num = b_B - l.z_T (acc[p-1]), so per cell
//   pivot = s_br - |l|^2,  beta_B = num / pivot,
//   beta_T = L^-T (z_T - l beta_B) = c_T - (L^-T l) beta_B
// with u = L^-T l an independent product (L^-1 packed by rows) that overlaps
// the reciprocal.  Same algebra as solve_cell, a shorter dependency chain and
// ~10 fewer FP64 operations; the pivot test is unchanged.
template <int P, bool SMEM = false>
__device__ __forceinline__ bool solve_cell_folded(const double* acc, const double* __restrict__ cx,
                                                  double* beta) {
  using L = CtxLayout<P>;
  constexpr int P1 = L::P1;
  double sq = 0.0;
#pragma unroll
  for (int a = 0; a < P1; ++a) sq = fma(acc[a], acc[a], sq);
  double u[P1 > 0 ? P1 : 1];
#pragma unroll
  for (int c = 0; c < P1; ++c) {
    double s = 0.0;
#pragma unroll
    for (int a = c; a < P1; ++a) s = fma(ctx_ld<SMEM>(cx + L::LINV + L::linv_idx(a, c)), acc[a], s);
    u[c] = s;
  }
  const double pivot = acc[P] - sq;
  const bool ok = !(pivot <= 0.0) && ctx_ld<SMEM>(cx + L::FLAG) == 0.0;
  double bb;
  if (P <= GWG_RCP_MAXP) {
    double r;
    r = rcp_newton(pivot);
    bb = acc[P1] * r;
    if (pivot < 0x1p-1022 && pivot > 0.0) bb = acc[P1] / pivot;  // subnormal: exact division
  } else {
    bb = acc[P1] / pivot;
  }
  beta[P1] = bb;
#pragma unroll
  for (int c = 0; c < P1; ++c) beta[c] = fma(-u[c], bb, ctx_ld<SMEM>(cx + L::CT + c));
  return ok;
}

// Runtime offsets of CtxLayout<p> (host launches of the trait-side kernels).
struct CtxOffsets {
  int z, flag, linv, ct, stride;
};
__host__ __device__ inline CtxOffsets ctx_offsets(int p) {
  const int p1 = p - 1, noff = p1 > 1 ? p1 * (p1 - 1) / 2 : 0;
  CtxOffsets o;
  o.z = p1 + noff;
  o.flag = 2 * p1 + noff;
  o.linv = o.flag + 1;
  o.ct = o.linv + p1 * (p1 + 1) / 2;
  o.stride = (o.ct + p1 + 1) & ~1;
  return o;
}

// Issue the TMA/bulk loads of global k-iteration g (tile g / kchunks of this
// CTA's static schedule, k-chunk g % kchunks) into its stage.
template <class Cfg>
__device__ __forceinline__ void issue_stage(const CUtensorMap* tmap_a, const CUtensorMap* tmap_q,
                                            const GridArgs& args,
                                            double* sA, double* sB, uint64_t* full,
                                            uint64_t* empty, int g, int total_iters,
                                            uint64_t pol_a, uint64_t pol_b, int group = 0) {
  if (g >= total_iters) return;
  constexpr int KO = Cfg::BK / 8;
  const int s = g % Cfg::STAGES;
  const int use = g / Cfg::STAGES;  // how many times this stage was filled before
  if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
  const int local_tile = g / args.kchunks;
  const int kc = g - local_tile * args.kchunks;
  const int tile = (blockIdx.x + local_tile * gridDim.x) * Cfg::GROUPS + group;
  const int tm = tile / args.tiles_t;
  const int tt = tile - tm * args.tiles_t;
  mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
  double* a_dst = sA + s * Cfg::SA_STAGE;
#pragma unroll
  for (int ko = 0; ko < KO; ++ko) {
    tma_load_2d(a_dst + ko * Cfg::BM * 8, tmap_a, (kc * KO + ko) * 8, tm * Cfg::BM, &full[s],
                pol_a);
    if (!Cfg::EXT)
      tma_load_2d(a_dst + Cfg::A_STAGE + ko * Cfg::BM * 8, tmap_q, (kc * KO + ko) * 8,
                  tm * Cfg::BM, &full[s], pol_a);
  }
  const double* bsrc = args.bops + size_t(tt) * size_t(args.np) * Cfg::NC * Cfg::BT +
                       size_t(kc) * Cfg::B_GSTAGE;
  if (Cfg::EXT) {  // the first P column blocks of every k-octet
#pragma unroll
    for (int ko = 0; ko < KO; ++ko)
      bulk_load(sB + s * Cfg::B_STAGE + ko * Cfg::NCS * Cfg::BT * 8,
                bsrc + ko * Cfg::NC * Cfg::BT * 8, uint32_t(Cfg::NCS * Cfg::BT * 8 * 8), &full[s],
                pol_b);
  } else {
    bulk_load(sB + s * Cfg::B_STAGE, bsrc, Cfg::B_BYTES, &full[s], pol_b);
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    gls_grid_kernel(const __grid_constant__ CUtensorMap tmap_a,
                    const __grid_constant__ CUtensorMap tmap_q, const GridArgs args) {
  if (gate_closed(args.gate, args.gate_codes)) return;
  constexpr int P = Cfg::P;
  constexpr int NC = Cfg::NCS;      // accumulated columns per cell
  constexpr int KO = Cfg::BK / 8;  // k-octets per stage
  constexpr int WO = Cfg::WM_OCT;
  constexpr int G = Cfg::GROUPS;
  extern __shared__ __align__(1024) double smem[];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // consumer warps 0..WARPS-1: group = warp / GWARPS would put a group on two
  // sub-partitions only; interleave instead so each SM sub-partition (warp % 4)
  // hosts one warp of every group.
  const bool is_producer_warp = Cfg::PRODUCER_WARP && warp >= Cfg::WARPS;
  const int group = is_producer_warp ? warp - Cfg::WARPS : (G == 1 ? 0 : (warp / 4) % G);
  const int lw = G == 1 ? warp : (warp % 4) + 4 * (warp / (4 * G));  // warp within group

  double* sA = smem + size_t(group) * Cfg::STAGES * (Cfg::SA_STAGE + Cfg::B_STAGE);
  double* sB = sA + Cfg::STAGES * Cfg::SA_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      smem + size_t(G) * Cfg::STAGES * (Cfg::SA_STAGE + Cfg::B_STAGE));
  uint64_t* full = bars + group * 2 * Cfg::STAGES;
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* go = bars + G * 2 * Cfg::STAGES;  // ping-pong phase gate

  const int ntiles = args.tiles_m * args.tiles_t;
  const int nsuper = (ntiles + G - 1) / G;
  const int my_super = blockIdx.x < nsuper ? (nsuper - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // this group's tiles: super tiles whose group-th member exists
  int my_tiles = my_super;
  if (my_super > 0 && (blockIdx.x + (my_super - 1) * gridDim.x) * G + group >= ntiles)
    --my_tiles;
  const int total_iters = my_tiles * args.kchunks;
  const bool producer = Cfg::PRODUCER_WARP ? (is_producer_warp && lane == 0) : threadIdx.x == 0;
  uint64_t pol_a = 0, pol_b = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < G * 2 * Cfg::STAGES; q += 2 * Cfg::STAGES)
      for (int s = 0; s < Cfg::STAGES; ++s) {
        mbar_init(&bars[q + s], 1);
        mbar_init(&bars[q + Cfg::STAGES + s], Cfg::GWARPS);
      }
    mbar_init(go, 1);
    fence_mbar_init();
  }
  if (producer) {
    pol_a = policy_evict_normal();  // SNP tile: re-read by the CTAs of its trait tiles
    pol_b = policy_evict_last();    // trait operands: L2-resident for the whole launch
  }
  __syncthreads();
  if (Cfg::PRODUCER_WARP) {
    if (is_producer_warp) {
      if (producer)
        for (int g = 0; g < (GWG_EXPERIMENT == 2 ? min(total_iters, Cfg::STAGES) : total_iters);
             ++g)
          issue_stage<Cfg>(&tmap_a, &tmap_q, args, sA, sB, full, empty, g, total_iters, pol_a,
                           pol_b, group);
      return;
    }
  } else if (producer) {
    for (int g = 0; g < Cfg::LOOKAHEAD; ++g)
      issue_stage<Cfg>(&tmap_a, &tmap_q, args, sA, sB, full, empty, g, total_iters, pol_a, pol_b);
  }

  const int wm = lw % Cfg::WARPS_M;
  const int wt = lw / Cfg::WARPS_M;
  const int half = args.kchunks / 2;
  if (G > 1 && group > 0 && my_tiles > 0) mbar_wait(go, 0);  // start half a tile late
  if (G > 1 && group == 0 && lw == 0 && lane == 0 && my_tiles == 0) mbar_arrive(go);
  int g = 0;
  for (int lt = 0; lt < my_tiles; ++lt) {
    const int tile = (blockIdx.x + lt * gridDim.x) * G + group;
    const int tm = tile / args.tiles_t;
    const int tt = tile - tm * args.tiles_t;

    double acc[WO][NC][2];
#pragma unroll
    for (int o = 0; o < WO; ++o)
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[o][c][0] = acc[o][c][1] = 0.0;

    for (int kc = 0; kc < args.kchunks; ++kc, ++g) {
      if (G > 1 && group == 0 && lt == 0 && kc == half && lw == 0 && lane == 0) mbar_arrive(go);
      // (in-loop producer only) thread 0 keeps LOOKAHEAD stages in flight; the
      // stage it refills was consumed two iterations ago (one slack stage).
      if (!Cfg::PRODUCER_WARP && producer)
        issue_stage<Cfg>(&tmap_a, &tmap_q, args, sA, sB, full, empty, g + Cfg::LOOKAHEAD,
                         total_iters, pol_a, pol_b);
      const int s = g % Cfg::STAGES;
      if (GWG_EXPERIMENT != 2 || g < Cfg::STAGES) mbar_wait(&full[s], (g / Cfg::STAGES) & 1);
      const double2* a2 = reinterpret_cast<const double2*>(sA + s * Cfg::SA_STAGE);
      const double2* q2 = a2 + Cfg::A_STAGE / 2;
      const double2* b2 = reinterpret_cast<const double2*>(sB + s * Cfg::B_STAGE);
#pragma unroll
      for (int ko = 0; ko < KO; ++ko) {
        double2 bf[NC], af[WO], sq[WO];
#pragma unroll
        for (int c = 0; c < NC; ++c)
          bf[c] = b2[((ko * NC + c) * Cfg::WARPS_T + wt) * 32 + lane];
#pragma unroll
        for (int o = 0; o < WO; ++o) {
          af[o] = a2[(ko * (Cfg::BM / 8) + wm * WO + o) * 32 + lane];
          if (!Cfg::EXT) sq[o] = q2[(ko * (Cfg::BM / 8) + wm * WO + o) * 32 + lane];
        }
        // even-k pass over every accumulator, then the odd-k pass: dependent
        // DMMAs on one accumulator are WO*NC instructions apart.
#pragma unroll
        for (int o = 0; o < WO; ++o) {
#pragma unroll
          for (int c = 0; c < P; ++c) dmma(acc[o][c], af[o].x, bf[c].x);
          if (!Cfg::EXT) dmma(acc[o][NC - 1], sq[o].x, bf[NC - 1].x);
        }
#pragma unroll
        for (int o = 0; o < WO; ++o) {
#pragma unroll
          for (int c = 0; c < P; ++c) dmma(acc[o][c], af[o].y, bf[c].y);
          if (!Cfg::EXT) dmma(acc[o][NC - 1], sq[o].y, bf[NC - 1].y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---------------- fused epilogue: bordered Cholesky + store -----------------
    using L = CtxLayout<P>;
    const uint64_t pol_out = policy_evict_first();
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = tt * Cfg::BT + wt * 8 + 2 * (lane & 3) + e;
      if (j >= args.t) continue;
      const double* cx = args.ctx + size_t(j) * L::STRIDE;
#pragma unroll
      for (int o = 0; o < WO; ++o) {
        const int64_t il = int64_t(tm) * Cfg::BM + (wm * WO + o) * 8 + (lane >> 2);
        if (il >= args.rows) continue;
        double cell[P + 1];
#pragma unroll
        for (int c = 0; c < NC; ++c) cell[c] = acc[o][c][e];
        if (Cfg::EXT) cell[P] = __ldcs(args.sbr + int64_t(j) * args.ld_s + il);
        double beta[P];
#if GWG_EXPERIMENT == 1
        bool ok = true;
#pragma unroll
        for (int c = 0; c < P; ++c) beta[c] = cell[c] + cell[P];
#else
        const bool ok = solve_cell<P>(cell, cx, beta);
#endif
        double* dst = args.out + (il * args.out_si + int64_t(j) * args.out_sj) * P;
        if (!ok) {
          atomicMin(args.err_key,
                    (unsigned long long)(int64_t(j) * args.m_total + args.i0 + il));
#pragma unroll
          for (int c = 0; c < P; ++c) beta[c] = __longlong_as_double(0x7ff8000000000000LL);
        }
#pragma unroll
        for (int c = 0; c < P; ++c) st_evict_first(dst + c, beta[c], pol_out);
      }
    }
  }
}

}  // namespace gwg
