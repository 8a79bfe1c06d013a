// linear_solve.cuh — second launch of the genotype split grid (grid_split.cuh):
// the p linear terms of every cell exactly on the int8 tensor cores, and the
// cell's bordered Cholesky solve in the same epilogue.
//
// GEMM view per CTA tile: M = 128 SNPs (A = int8 genotype codes, K-major),
// N = 8 slices x RB rows of W (B, K-major), K = samples; int32 accumulators in
// TMEM, double-buffered (the TMA producer / MMA issuer / TMEM code is shared
// with rotate_i8_kernel); CTA pairs (cluster of 2) take SNP tiles 2u, 2u+1 of
// the same W rows and multicast halves of the W-slice tile.  W is laid out per
// tile of KT traits, each trait's p columns padded to P8 (a power of two <= 8,
// else a multiple of 8) so that a trait's columns are one aligned tcgen05.ld.
//
// Epilogue (thread = SNP row): 16 warps for p <= 16 (two per accumulator
// buffer and TMEM lane quarter, each half of a tile's cells), else 8 (one per
// buffer and quarter, all cells).  Per cell (i, j) the p linear terms
// x_i^T W_{j,c} are recombined exactly from the eight slice products
// (i8_recombine, one rounding), S_BR[j][i] comes from gls_sbr_kernel
// (prefetched before the accumulator wait), and the bordered Cholesky —
// solve_cell<P> as in the all-FP64 kernel, or solve_cell_inv<P> with the
// precomputed L^-1 for p >= 9 — produces b_ij, which leaves through a
// 128B-swizzled staging tile and an evict_first TMA store (numpy layout) or
// direct stores (stream layout).  Failed cells: NaN + the min error key,
// exactly like gls_grid_kernel.
#pragma once

#include "grid_kernel.cuh"
#include "i8_core.cuh"


namespace gwg {

// Timing ablations only (never in a shipped build): 1 = no result stores,
// 2 = no S_BR loads, 3 = no solve, 4 = neither solve nor stores, 5 = 4 and
// no S_BR loads and a plain sum for the recombination, 6 = 5 without the
// TMEM loads, 7 = every TMA result store to the same 4 KB (no DRAM writes).
#ifndef LIN_EXPERIMENT
#define LIN_EXPERIMENT 0
#endif

#ifndef LIN_STREAM_HALF
#define LIN_STREAM_HALF 0  // per-group boxes measured slower at c1 (2.37 vs 2.34 ms)
#endif
#ifndef LIN_STG_RECOMPUTE
#define LIN_STG_RECOMPUTE 0
#endif
#ifndef LIN_STORE_EXP
#define LIN_STORE_EXP 0
#endif

#ifndef LIN_TRACE
#define LIN_TRACE 0
#endif

#ifndef LIN_WIDE_MAXP
#define LIN_WIDE_MAXP 16
#endif

#ifndef LIN_EARLY_RELEASE
#define LIN_EARLY_RELEASE 1
#endif

// W folded with L_j^-1 on the trait side (fold_w_kernel): the epilogue runs
// solve_cell_folded (the engine folds W exactly when this is on)
#ifndef LIN_FOLD
#define LIN_FOLD 1
#endif

// Register reallocation between warpgroups (setmaxnreg): the producer / MMA /
// context warpgroup drops to 40 registers and the epilogue warpgroups rise to
// LIN_MAXNREG (0 = off), with deeper per-warp interleaving (LIN_GMAX cells
// solved together, LIN_PAIR cells per TMEM round trip) in that budget
#ifndef LIN_MAXNREG
#define LIN_MAXNREG 0
#endif
#ifndef LIN_GMAX
#define LIN_GMAX 0
#endif
#ifndef LIN_PAIR
#define LIN_PAIR 0
#endif

// S_BR: the context warp prefetches each tile's S_BR rows into L2 (bulk
// prefetch) and the epilogue loads them after the TMEM release, instead of
// holding a register prefetch from HBM across the accumulator wait
// (measured slower at c1: 2.68 vs 2.45 ms; off)
#ifndef LIN_SBR_L2PF
#define LIN_SBR_L2PF 0
#endif
#ifndef LIN_SBR_LATE  // with the L2 prefetch: load after the release (1) or before the wait (0)
#define LIN_SBR_LATE 1
#endif

// Per-tile trait contexts and W-row scales staged in shared memory by bulk
// copies (warp 2) instead of per-cell __ldg / shuffles in the epilogue.
// producer and MMA loops run warp-collectively (I8Tile WS)
#ifndef LIN_WS
#define LIN_WS 1
#endif

#ifndef LIN_WS_MMA2  // warp-collective issue for the pair MMA too (measured slower at c2)
#define LIN_WS_MMA2 0
#endif

#ifndef LIN_CTX_SMEM
#define LIN_CTX_SMEM 1
#endif
#ifndef LIN_CTX_SLOTS  // context staging slots (>= the 2 accumulator buffers)
#define LIN_CTX_SLOTS 4
#endif

// p % 4 == 0: results leave by direct 256-bit stores from registers (any
// layout; no staging tiles), and the shared memory that frees holds each
// tile's S_BR rows, staged by one TMA box per tile from the context warp, and
// a fourth operand stage
#ifndef LIN_NOSTAGE
#define LIN_NOSTAGE 0  // measured at c1: neutral with S_BR per cell and 3 stages, slower otherwise (off)
#endif
#ifndef LIN_SBR_TMA  // NOSTAGE: S_BR staged by TMA (1) or loaded per cell as before (0)
#define LIN_SBR_TMA 1
#endif
#ifndef LIN_NOSTAGE_DEEP  // NOSTAGE: one more operand stage
#define LIN_NOSTAGE_DEEP 1
#endif

template <int P, int CL = 1>
struct LinCfg {
  static constexpr int P8 = P <= 1 ? 1 : P <= 2 ? 2 : P <= 4 ? 4 : P <= 8 ? 8 : (P + 7) / 8 * 8;
  static constexpr int KT = 32 / P8 >= 1 ? 32 / P8 : 1;  // traits per tile
  static constexpr int RB = KT * P8;                      // W rows per tile (24 or 32)
  // WIDE (p <= 16): 16 epilogue warps (4 per TMEM lane quarter: 2 per
  // accumulator buffer, each doing half of a tile's cells; 96 registers) with
  // 3 operand stages — the epilogue is latency-bound, so more warps beat
  // deeper operand buffering; otherwise (the O(p^2) solve needs registers)
  // 8 epilogue warps (2 per quarter, all cells of alternate tiles) and 4
  // stages.  One 4 KB staging tile per epilogue warp.
  static constexpr bool WIDE = P <= LIN_WIDE_MAXP;  // measured: p=4 3.15 -> 2.83 ms, p=12 8.56 -> 7.95
  static constexpr int EPI = WIDE ? 16 : 8;
  static constexpr int ACC = 2;                           // TMEM accumulator buffers
  static constexpr int HMAX = EPI / 4 / ACC;              // warps per quarter and buffer
  static constexpr int HALVES = KT >= HMAX ? HMAX : 1;    // warps splitting one tile
  static constexpr int CELLS = KT / HALVES;               // cells per warp per tile
  static constexpr int CW = P8 < 8 ? P8 : 8;              // TMEM columns per load
  static constexpr int ROW = CELLS * P;                   // results per warp row per tile
  static constexpr int CHUNK = 16;                        // doubles per swizzled TMA row (128 B)
  static constexpr bool TMA_OUT = ROW % CHUNK == 0;       // whole 128-byte chunks
  // other even rows of <= 32 doubles leave through one unswizzled TMA box
  // {ROW, 32} per warp and tile (direct stores cost p = 12 2.8 of 7.8 ms and
  // c4 8.7 of 37.9 ms); rows above 16 doubles need an 8 KB staging tile
  // (an odd row's last double is stored directly: a box row is a multiple of
  // 16 bytes)
  static constexpr bool TMA_ROW = !TMA_OUT && ROW >= 2 && ROW <= 33;
  // stream order ((j*ldo + i)*p, the reference's ResultTile / result-stream
  // layout): a warp's results are, per trait, 32 SNPs x p contiguous doubles;
  // staged [cell][lane*p + c] and stored as one TMA box {32p, CELLS}
  static constexpr bool STREAM_TMA = 32 * P <= 256 && CELLS * 32 * P * 8 <= 4096;
  // stream boxes per group of cells (GROUP rows) instead of per tile (CELLS rows)
  static constexpr bool STREAM_HALF = LIN_STREAM_HALF != 0;
  // stream order by direct 256-bit stores from registers (use_tma = 3): a
  // lane's p results of a cell are p/4 aligned 32-byte pieces, a warp's cell
  // 32p contiguous doubles — no staging, no proxy fence, no TMA store
  static constexpr bool STREAM_STG = P % 4 == 0;
  static constexpr int BW = ROW & ~1;                     // doubles per TMA box row
  static constexpr bool NOSTAGE = LIN_NOSTAGE != 0 && LIN_CTX_SMEM != 0 && P % 4 == 0;
  static constexpr int OUT_BUFS = NOSTAGE ? 0 : TMA_ROW && BW * 8 * 32 > 4096 ? 2 : 1;
  // CL = 4: CTA pairs running one cta_group::2 MMA, half of B per CTA
  // (I8Tile MMA2; 32-row W tiles only)
  static constexpr bool MMA2 = CL == 4;
  static_assert(!MMA2 || RB == 32, "pair MMA on 32-row W tiles");
  static constexpr bool DEEP = NOSTAGE && LIN_NOSTAGE_DEEP;
  static constexpr bool SBR_TMA = NOSTAGE && LIN_SBR_TMA;
#ifndef LIN_STAGES  // timing override of the operand stages (0 = the default below)
#define LIN_STAGES 0
#endif
  static constexpr int STAGES_0 = LIN_STAGES > 0 ? LIN_STAGES
                                  : MMA2 ? (WIDE && !DEEP ? 5 : 6) : WIDE && !DEEP ? 3 : 4;
  static constexpr uint32_t STAGE_B = MMA2 ? 128 * 128 + 7 * RB * 64 : 128 * 128 + 8 * RB * 128;
  // shared-memory context staging, per accumulator buffer: the tile's KT trait
  // contexts (CtxLayout, contiguous in global memory) and RB W-row scales,
  // then the ctx_full / ctx_empty mbarriers
  static constexpr bool CTX_SMEM = LIN_CTX_SMEM != 0;
  static constexpr int CTX_DOUBLES = KT * CtxLayout<P>::STRIDE;
  static constexpr uint32_t CTX_BYTES = CTX_DOUBLES * 8;
  // context slots: tile lt uses slot lt % NCTX; with NCTX > ACC the context
  // warp loads a tile's contexts NCTX - ACC tiles ahead of its epilogue
  // instead of right after the same warps finished the tile before it
  static constexpr int NCTX = LIN_CTX_SLOTS > ACC ? LIN_CTX_SLOTS : ACC;
  static_assert(NCTX % ACC == 0, "a warp's tiles cycle through the slots in order");
  static constexpr uint32_t SCALE_OFF = NCTX * CTX_BYTES;
  // NOSTAGE: per accumulator buffer the tile's S_BR box [KT traits][BM SNPs]
  static constexpr uint32_t SBR_BYTES = SBR_TMA ? KT * 128 * 8 : 0;
  static constexpr uint32_t SBR_OFF = (SCALE_OFF + NCTX * RB * 8 + 127) / 128 * 128;
  static constexpr uint32_t BAR_OFF = SBR_OFF + NCTX * SBR_BYTES;
  static constexpr uint32_t EXTRA = CTX_SMEM ? BAR_OFF + 2 * NCTX * 8 : 0;
  static constexpr size_t FIXED_B = size_t(EPI) * OUT_BUFS * 4096 + (EXTRA + 15) / 16 * 16 + 1280;
  static constexpr int STAGES = size_t(STAGES_0) * STAGE_B + FIXED_B <= 227 * 1024 ? STAGES_0
                                : size_t(STAGES_0 - 1) * STAGE_B + FIXED_B <= 227 * 1024
                                    ? STAGES_0 - 1
                                    : STAGES_0 - 2;
  // CL = 3: CTA pairs along the trait axis sharing (multicasting) the SNP tile
  // CL = 5: 2 x 2 clusters multicasting halves of both operands
  // warp-collective issue except for the pair MMA (measured, see i8_core.cuh)
  using Tile = I8Tile<RB, STAGES, OUT_BUFS, EPI, CL == 5 ? 4 : CL >= 2 ? 2 : 1,
                      CL == 3 ? 1 : CL == 5 ? 2 : 0, EXTRA, MMA2,
                      LIN_WS != 0 && (!MMA2 || LIN_WS_MMA2 != 0)>;
  static_assert(Tile::ACC_BUFS == ACC && Tile::OUT_Q == CHUNK, "tile geometry");
  // cells solved together (independent chains; KT is a power of two or 1)
  static constexpr int GMAX = LIN_GMAX > 0 && P <= 4 ? LIN_GMAX
                              : WIDE ? (P <= 4 ? 2 : 1) : (P <= 4 ? 4 : (P <= 16 ? 2 : 1));
  static constexpr int GROUP = CELLS < GMAX ? CELLS : GMAX;
  // EARLY: recombine every cell of the warp's tile share from TMEM first,
  // release the accumulator buffer, then solve and store: the MMA of tile
  // lt + ACC waits only for the recombination, not for the solves
  static constexpr bool EARLY = LIN_EARLY_RELEASE != 0 && CELLS * P <= 16;
  static constexpr int PAIR = LIN_PAIR > 0 && P <= 4 && CELLS % LIN_PAIR == 0 ? LIN_PAIR
                              : !EARLY && GROUP >= 2 && P8 <= 8 ? 2 : 1;  // cells per TMEM round trip
  // large p: triangular solves as products with L^-1 (independent dot
  // products instead of serial substitution chains)
#ifndef LIN_INV_MINP
#define LIN_INV_MINP 9
#endif
  static constexpr bool INV_SOLVE = P >= LIN_INV_MINP;
};

struct LinArgs {
  const double* scale;  // sigma per (padded) W row
  const double* sbr;    // S_BR[j * ld_s + i] from gls_sbr_kernel
  int64_t ld_s;
  const double* ctx;    // per-trait contexts (CtxLayout<P>)
  double* out;
  int64_t out_si;       // cell strides of out
  int64_t out_sj;
  int32_t use_tma;      // out through tmap_out: 1 numpy layout, 2 stream layout
  int32_t t;
  int64_t rows;
  int64_t i0;
  int64_t m_total;
  int32_t tiles_m;
  int32_t tiles_r;      // ceil(t / KT)
  int32_t kstages;
  int32_t b_resident;   // sliced operand fits L2: keep it resident
  unsigned long long* err_key;
  const unsigned long long* gate = nullptr;  // GWG_SNP_AUTO path gate (gate_closed)
  int32_t gate_codes = 0;
  int32_t raster = 0;   // I8Sched raster: 1 = trait tiles fastest (numpy-order results)
};

#if LIN_TRACE
// Timing trace (never in a shipped build): CTA 0, the 8 epilogue warps of
// TMEM lane quarter 0 and 1... (warps 4..11), first 48 of their tiles:
// [0] before the acc_full wait, [1] after it, [2] TMEM released, [3] tile done.
__device__ long long g_lin_trace[16][48][4];
__device__ long long g_lin_t0;
#endif

template <int P, int CL>
__global__ void __launch_bounds__(LinCfg<P, CL>::Tile::THREADS, 1)
    linear_solve_kernel(const __grid_constant__ CUtensorMap tmap_x,
                        const __grid_constant__ CUtensorMap tmap_w,
                        const __grid_constant__ CUtensorMap tmap_out, const LinArgs a,
                        const __grid_constant__ CUtensorMap tmap_wh) {
  if (gate_closed(a.gate, a.gate_codes)) return;
  using L = LinCfg<P, CL>;
  using C = typename L::Tile;
  using CX = CtxLayout<P>;
  extern __shared__ __align__(1024) unsigned char smem_ls[];
  const I8Smem<C> sm(smem_ls);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const I8Sched<C> sch(a.tiles_m, a.tiles_r, a.raster);
  const int my_tiles = sch.my_tiles;
  double* const ctx_sm = reinterpret_cast<double*>(sm.extra);
  double* const scale_sm = reinterpret_cast<double*>(sm.extra + L::SCALE_OFF);
  double* const sbr_sm = reinterpret_cast<double*>(sm.extra + L::SBR_OFF);
  uint64_t* const ctx_full = reinterpret_cast<uint64_t*>(sm.extra + L::BAR_OFF);
  uint64_t* const ctx_empty = ctx_full + L::NCTX;
  if (L::CTX_SMEM && threadIdx.x == 0) {  // fenced and published by i8_setup
    for (int b = 0; b < L::NCTX; ++b) {
      mbar_init(&ctx_full[b], 1);
      mbar_init(&ctx_empty[b], 4 * L::HMAX);
    }
  }
  // HMAX warps per quarter release each tile's buffer
  const uint32_t tmem_base = i8_setup<C>(sm, warp, 4 * L::HMAX);
#if LIN_MAXNREG
  if (warp < 4)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
  else
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(LIN_MAXNREG) : "memory");
#endif

  if (warp == 0) {
    if (C::WS || lane == 0)
      i8_produce<C>(sm, &tmap_x, &tmap_w, sch, a.kstages, a.b_resident != 0, &tmap_wh);
  } else if (warp == 1) {
    if (C::WS || lane == 0) i8_mma<C>(sm, tmem_base, my_tiles, a.kstages);
  } else if (warp == 2) {
    // context producer: tile lt's KT trait contexts and RB W-row scales into
    // the slot of its accumulator buffer once the epilogue of tile lt - ACC
    // released it (two bulk copies completing on ctx_full)
    if (L::CTX_SMEM && lane == 0) {
      const uint64_t pol = policy_evict_last();
      for (int lt = 0; lt < my_tiles; ++lt) {
        const int buf = lt % L::NCTX;
        if (lt >= L::NCTX) mbar_wait(&ctx_empty[buf], uint32_t((lt / L::NCTX) - 1) & 1);
        int tm, tr;
        sch.coords(lt, tm, tr);
        const int j0 = tr * L::KT;
        // a CTA pair along the trait axis (CL = 3) may get a tile past the
        // last trait: nothing to copy, the phase still completes
        const int nt = tr < a.tiles_r ? min(L::KT, a.t - j0) : 0;
        const uint32_t cbytes = uint32_t(nt) * CX::STRIDE * 8;
        mbar_arrive_expect_tx(&ctx_full[buf], nt > 0 ? cbytes + C::RB * 8 + L::SBR_BYTES : 0);
        if (nt > 0) {
          bulk_load(ctx_sm + buf * L::CTX_DOUBLES, a.ctx + int64_t(j0) * CX::STRIDE, cbytes,
                    &ctx_full[buf], pol);
          bulk_load(scale_sm + buf * C::RB, a.scale + int64_t(tr) * C::RB, C::RB * 8,
                    &ctx_full[buf], pol);
          // S_BR rows [j0, +KT) x SNPs [tm BM, +BM) (tmap_out is the S_BR map
          // here; zero-filled past either edge, the full box still counts)
          if (L::SBR_TMA)
            tma_load_2d(sbr_sm + buf * (L::SBR_BYTES / 8), &tmap_out, tm * C::BM, j0,
                        &ctx_full[buf], policy_evict_first());
        }
        if (LIN_SBR_L2PF) {  // this tile's S_BR rows [j][tm*BM, +BM) into L2
          const int64_t i_lo = int64_t(tm) * C::BM;
          const int64_t cnt = min(int64_t(C::BM), a.rows - i_lo);
          const uint32_t bytes = uint32_t((cnt + 1) & ~int64_t(1)) * 8;  // ld_s is even
          for (int u = 0; u < nt; ++u)
            bulk_prefetch_l2(a.sbr + int64_t(j0 + u) * a.ld_s + i_lo, bytes);
        }
      }
    }
  } else if (warp >= 4) {
    // warp w owns TMEM lane quarter w % 4; the two warps of a quarter take
    // alternate tiles (= alternate accumulator buffers), each doing all KT
    // cells of its tile, so two tiles' epilogues are in flight per quarter.
    // (Warps per quarter must equal the number of accumulator buffers: each
    // warp then waits on one buffer's acc_full phases strictly in order — a
    // third warp per quarter could run two phases ahead and alias the parity.)
    const int ew = warp - 4;
    const int qd = warp & 3;
    const int h = (ew >> 2) % L::ACC;      // accumulator buffer (tile index mod ACC) of this warp
    const int hf = (ew >> 2) / L::ACC;     // which share of the tile's cells (HMAX > 1)
    const int cell0 = hf * L::CELLS;
    const bool active = cell0 < L::KT;
    unsigned char* stg = sm.staging + ew * C::OUT_BYTES;
    const uint64_t pol_out = policy_evict_first();
    int nchunk = 0;  // result chunks this warp has stored (staging tile = nchunk & 1)
    for (int lt = h; lt < my_tiles; lt += L::ACC) {
      const int buf = lt % L::ACC;
      const uint32_t par = uint32_t(lt / L::ACC) & 1;
      const int cslot = lt % L::NCTX;                         // context slot
      const uint32_t cpar = uint32_t(lt / L::NCTX) & 1;
      int tm, tr;
      sch.coords(lt, tm, tr);
      const int64_t il = int64_t(tm) * C::BM + qd * 32 + lane;
      const bool iv = il < a.rows;
      const int j0 = tr * L::KT;  // first trait of the tile
      if (!active) {  // KT = 1 under WIDE: nothing to do but keep the buffer protocol
        mbar_wait(&sm.acc_full[buf], par);
        if (L::CTX_SMEM) mbar_wait(&ctx_full[cslot], cpar);
        __syncwarp();
        if (lane == 0) {
          i8_acc_release<C>(sm, buf);
          if (L::CTX_SMEM) mbar_arrive(&ctx_empty[cslot]);
        }
        continue;
      }
      constexpr bool SBR_LATE = L::CTX_SMEM && L::EARLY && LIN_SBR_L2PF && LIN_SBR_LATE;
      double sbr[L::CELLS];
      auto load_sbr = [&]() {
#pragma unroll
        for (int cc = 0; cc < L::CELLS; ++cc) {
          const int j = j0 + cell0 + cc;
          if (LIN_EXPERIMENT == 2 || LIN_EXPERIMENT >= 5)
            sbr[cc] = 1e6 + lane;
          else
            sbr[cc] = (iv && j < a.t) ? __ldcs(a.sbr + int64_t(j) * a.ld_s + il) : 0.0;
        }
      };
      if (!SBR_LATE && !L::SBR_TMA) load_sbr();
      // without the staged copy, lane r holds the slice scale (sigma 2^-55) of
      // the tile's W row r (RB <= 32), shuffled to the recombination below
      const double sc_lane = !L::CTX_SMEM && lane < C::RB ? __ldg(a.scale + tr * C::RB + lane) : 0.0;
      const double* const cx_tile = ctx_sm + cslot * L::CTX_DOUBLES;
      const double* const sc_tile = scale_sm + cslot * C::RB;
#if LIN_TRACE
      const int tix = (lt - h) / L::ACC;
      const bool tr_on = blockIdx.x == 0 && lane == 0 && tix < 48;
      if (tr_on) g_lin_trace[ew][tix][0] = clock64();
#endif
      mbar_wait(&sm.acc_full[buf], par);
      if (L::CTX_SMEM) mbar_wait(&ctx_full[cslot], cpar);
#if LIN_TRACE
      if (tr_on) g_lin_trace[ew][tix][1] = clock64();
#endif
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(qd * 32) << 16) + uint32_t(buf * C::BN);
      const bool tma = L::TMA_OUT && a.use_tma == 1;
      // GROUP cells at a time: recombine their linear terms from TMEM (PAIR
      // cells per TMEM round trip), release TMEM after the last group, then
      // solve the group's independent cells together and store them.
      auto recombine = [&](int cb, int count, double(*dst)[P]) {
#pragma unroll
        for (int u0 = 0; u0 < count; u0 += L::PAIR) {
#pragma unroll
          for (int c0 = 0; c0 < P; c0 += L::CW) {
            int32_t v[L::PAIR][C::SLICES][L::CW];
#pragma unroll
            for (int u = 0; u < L::PAIR; ++u)
#pragma unroll
              for (int sl = 0; sl < C::SLICES; ++sl) {
                if (LIN_EXPERIMENT == 6) {
#pragma unroll
                  for (int r = 0; r < L::CW; ++r) v[u][sl][r] = lane + sl + r + u;
                } else {
                  tmem_ldw<L::CW>(taddr + uint32_t(sl * C::RB + (cb + u0 + u) * L::P8 + c0),
                                  v[u][sl]);
                }
              }
            if (LIN_EXPERIMENT != 6) tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < L::PAIR; ++u)
#pragma unroll
              for (int r = 0; r < L::CW; ++r) {
                if (c0 + r < P) {
                  const int wrow = (cb + u0 + u) * L::P8 + c0 + r;
                  const double sc = L::CTX_SMEM ? sc_tile[wrow]
                                                : __shfl_sync(0xffffffffu, sc_lane, wrow);
                  if (LIN_EXPERIMENT == 5)
                    dst[u0 + u][c0 + r] = double(v[u][0][r] + v[u][1][r] + v[u][2][r] +
                                                 v[u][3][r] + v[u][4][r] + v[u][5][r] +
                                                 v[u][6][r]) * sc;
                  else
                    dst[u0 + u][c0 + r] = i8_recombine(v[u][0][r], v[u][1][r], v[u][2][r],
                                                       v[u][3][r], v[u][4][r], v[u][5][r],
                                                       v[u][6][r], sc);
                }
              }
          }
        }
      };
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) i8_acc_release<C>(sm, buf);  // TMEM buffer free for tile lt + ACC
      };
      double lin_all[L::EARLY ? L::CELLS : 1][P];
      if constexpr (L::EARLY) {
        recombine(cell0, L::CELLS, lin_all);
        release();
        if (SBR_LATE) load_sbr();
#if LIN_TRACE
        if (tr_on) g_lin_trace[ew][tix][2] = clock64();
#endif
      }
#pragma unroll
      for (int g0 = 0; g0 < L::CELLS; g0 += L::GROUP) {
        double lin[L::GROUP][P];
        if constexpr (L::EARLY) {
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u)
#pragma unroll
            for (int c = 0; c < P; ++c) lin[u][c] = lin_all[g0 + u][c];
        } else {
          recombine(cell0 + g0, L::GROUP, lin);
          if (g0 + L::GROUP >= L::CELLS) {
            release();
#if LIN_TRACE
            if (tr_on) g_lin_trace[ew][tix][2] = clock64();
#endif
          }
        }
        double beta[L::GROUP][P];
        bool ok[L::GROUP];
#pragma unroll
        for (int u = 0; u < L::GROUP; ++u) {
          const int j = j0 + cell0 + g0 + u;
          const bool cv = j < a.t && iv;
          double cell[P + 1];
#pragma unroll
          for (int c = 0; c < P; ++c) cell[c] = lin[u][c];
          cell[P] = L::SBR_TMA ? sbr_sm[(cslot * L::KT + cell0 + g0 + u) * 128 + qd * 32 + lane]
                               : sbr[g0 + u];
          const double* cx = L::CTX_SMEM ? cx_tile + (cell0 + g0 + u) * CX::STRIDE
                                         : a.ctx + size_t(cv ? j : 0) * CX::STRIDE;
          if (LIN_EXPERIMENT >= 3) {
#pragma unroll
            for (int c = 0; c < P; ++c) beta[u][c] = cell[c] + cell[P];
            ok[u] = true;
          } else {
            ok[u] = (LIN_FOLD ? solve_cell_folded<P, L::CTX_SMEM>(cell, cx, beta[u])
                     : L::INV_SOLVE ? solve_cell_inv<P, L::CTX_SMEM>(cell, cx, beta[u])
                                    : solve_cell<P, L::CTX_SMEM>(cell, cx, beta[u])) ||
                    !cv;
          }
        }
#pragma unroll
        for (int u = 0; u < L::GROUP; ++u) {
          if (!ok[u]) {
            const int j = j0 + cell0 + g0 + u;
            atomicMin(a.err_key, (unsigned long long)(int64_t(j) * a.m_total + a.i0 + il));
#pragma unroll
            for (int c = 0; c < P; ++c) beta[u][c] = __longlong_as_double(0x7ff8000000000000LL);
          }
        }
        if (LIN_EXPERIMENT == 1 || LIN_EXPERIMENT >= 4) {
          // keep the results live without storing them
          double acc = 0.0;
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u)
#pragma unroll
            for (int c = 0; c < P; ++c) acc += beta[u][c];
          if (acc == 1.2345e300) a.out[il] = acc;
        } else if (L::NOSTAGE) {
          // any layout: a cell's p doubles are p/4 aligned 32-byte pieces
          // (use_tma = 3) or, for a base not 32-byte aligned, plain stores
          if (iv) {
#pragma unroll
            for (int u = 0; u < L::GROUP; ++u) {
              const int j = j0 + cell0 + g0 + u;
              if (j >= a.t) continue;
              double* dst = a.out + (il * a.out_si + int64_t(j) * a.out_sj) * P;
              // timing only (LIN_STORE_EXP): 1 = every other cell stored (half the
              // bytes), 2 = the same stores folded into a 16 MB window (L2-resident,
              // no DRAM writes)
              if (LIN_STORE_EXP == 1 && (u & 1)) continue;
              if (LIN_STORE_EXP == 2)
                dst = a.out + ((il * a.out_si + int64_t(j) * a.out_sj) * P) % (int64_t(1) << 21);
              if (a.use_tma == 3) {
#pragma unroll
                for (int c = 0; c < P; c += 4)
                  st4_policy(dst + c, beta[u][c], beta[u][c + 1], beta[u][c + 2], beta[u][c + 3],
                             pol_out);
              } else {
#pragma unroll
                for (int c = 0; c < P; ++c) st_evict_first(dst + c, beta[u][c], pol_out);
              }
            }
          }
        } else if (L::STREAM_STG && a.use_tma == 3) {
          if (iv) {
#pragma unroll
            for (int u = 0; u < L::GROUP; ++u) {
              const int j = j0 + cell0 + g0 + u;
              if (j >= a.t) continue;
              double* dst = a.out + (il + int64_t(j) * a.out_sj) * P;
#pragma unroll
              for (int c = 0; c < P; c += 4)
                st4_policy(dst + c, beta[u][c], beta[u][c + 1], beta[u][c + 2], beta[u][c + 3],
                           pol_out);
            }
          }
        } else if (L::STREAM_TMA && a.use_tma == 2 && L::STREAM_HALF) {
          // one box {32p, GROUP} per group of cells, the staging tile used as
          // CELLS / GROUP slots in turn: a slot is rewritten only after the
          // store issued CELLS / GROUP groups earlier has read it, so the wait
          // is for an older store than the one just issued
          constexpr int SLOTS = L::CELLS / L::GROUP;
          if (lane == 0) {
            if constexpr (SLOTS >= 2)
              bulk_wait_read1();
            else
              bulk_wait_read0();
          }
          __syncwarp();
          double* rowp = reinterpret_cast<double*>(stg) + (g0 / L::GROUP) * (L::GROUP * 32 * P);
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u)
#pragma unroll
            for (int c = 0; c < P; ++c) rowp[(u * 32 + lane) * P + c] = beta[u][c];
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0)
            tma_store_2d(&tmap_out, rowp, (tm * C::BM + qd * 32) * P, j0 + cell0 + g0);
        } else if (L::STREAM_TMA && a.use_tma == 2) {
          if (g0 == 0) {
            if (lane == 0) bulk_wait_read0();  // the previous tile's store has read it
            __syncwarp();
          }
          unsigned char* stg_now = stg;
          if (LIN_STG_RECOMPUTE) {  // recomputed here instead of kept live (ptxas spilled it)
            uint32_t tid;
            asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
            stg_now = sm.staging + ((tid >> 5) - 4) * C::OUT_BYTES;
          }
          double* rowp = reinterpret_cast<double*>(stg_now);
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u)
#pragma unroll
            for (int c = 0; c < P; ++c) rowp[((g0 + u) * 32 + lane) * P + c] = beta[u][c];
          if (g0 + L::GROUP >= L::CELLS) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0)
              tma_store_2d(&tmap_out, stg_now, (tm * C::BM + qd * 32) * P, j0 + cell0);
          }
        } else if (tma) {
          // flat index f = (g0+u)*P + c of this row; 128-byte chunks of 16
          // doubles, 16-byte units XOR-swizzled by row (SWIZZLE_128B), one
          // TMA store per chunk
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u)
#pragma unroll
            for (int c = 0; c < P; ++c) {
              const int f = (g0 + u) * P + c;
              unsigned char* tile_buf =
                  stg + (C::OUT_BUFS == 2 ? ((nchunk + f / L::CHUNK) & 1) * C::OUT_TILE : 0);
              if (f % L::CHUNK == 0) {  // starting a chunk: its staging tile must be free
                if (lane == 0) {
                  if (C::OUT_BUFS == 2)
                    bulk_wait_read1();
                  else
                    bulk_wait_read0();
                }
                __syncwarp();
              }
              const int q = (f % L::CHUNK) >> 1;
              *reinterpret_cast<double*>(tile_buf + lane * 128 + ((q ^ (lane & 7)) << 4) +
                                         (f & 1) * 8) = beta[u][c];
              if (f % L::CHUNK == L::CHUNK - 1) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  if (LIN_EXPERIMENT == 7)  // timing only: the same instructions, one 4 KB target
                    tma_store_2d(&tmap_out, tile_buf, 0, 0);
                  else
                    tma_store_2d(&tmap_out, tile_buf,
                                 (j0 + cell0) * P + (f / L::CHUNK) * L::CHUNK,
                                 tm * C::BM + qd * 32);
                }
              }
            }
        } else if (L::TMA_ROW && a.use_tma == 1) {
          // the warp's ROW results per SNP row, unswizzled [lane][ROW] in the
          // staging tile, one TMA box {ROW, 32} after the tile's last group
          if (g0 == 0) {
            if (lane == 0) bulk_wait_read0();  // the previous tile's store has read it
            __syncwarp();
          }
          // an odd row keeps one double out of the box: the last one when the
          // row starts 16-byte aligned, else the first (the box start must be)
          const int shift = (L::ROW & 1) ? (((j0 + cell0) * P) & 1) : 0;
          double* row = reinterpret_cast<double*>(stg) + lane * L::BW;
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u)
#pragma unroll
            for (int c = 0; c < P; ++c) {
              const int f = (g0 + u) * P + c - shift;
              if (f >= 0 && f < L::BW) {
                row[f] = beta[u][c];
              } else if (iv && j0 + cell0 + g0 + u < a.t) {  // odd row: the double left out
                st_evict_first(
                    a.out + (il * a.out_si + int64_t(j0 + cell0 + g0 + u) * a.out_sj) * P + c,
                    beta[u][c], pol_out);
              }
            }
          if (g0 + L::GROUP >= L::CELLS) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0)
              tma_store_2d(&tmap_out, stg, (j0 + cell0) * P + shift, tm * C::BM + qd * 32);
          }
        } else if (iv) {
#pragma unroll
          for (int u = 0; u < L::GROUP; ++u) {
            const int j = j0 + cell0 + g0 + u;
            if (j >= a.t) continue;
            double* dst = a.out + (il * a.out_si + int64_t(j) * a.out_sj) * P;
#pragma unroll
            for (int c = 0; c < P; ++c) st_evict_first(dst + c, beta[u][c], pol_out);
          }
        }
      }
      if (L::CTX_SMEM) {  // this warp is done with the tile's contexts and scales
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctx_empty[cslot]);
      }
      if (tma) nchunk += L::ROW / L::CHUNK;
#if LIN_TRACE
      if (tr_on) g_lin_trace[ew][tix][3] = clock64();
#endif
    }
    if (lane == 0) bulk_wait0();
  }
  i8_teardown<C>(tmem_base, warp);
#if LIN_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0 && P == 4) {
    for (int w = 0; w < 16; ++w)
      for (int i = 0; i < 48; ++i)
        printf("LTR %d %d %lld %lld %lld %lld\n", w, i, g_lin_trace[w][i][0], g_lin_trace[w][i][1],
               g_lin_trace[w][i][2], g_lin_trace[w][i][3]);
  }
#endif
}

template <int P, int CL>
cudaError_t launch_linear_solve(const CUtensorMap& tx, const CUtensorMap& tw,
                                const CUtensorMap& tout, const LinArgs& a, int sms,
                                cudaStream_t s, const CUtensorMap& twh) {
  using C = typename LinCfg<P, CL>::Tile;
  const int64_t units = C::PAIR_AXIS == 2 ? int64_t((a.tiles_m + 1) / 2) * ((a.tiles_r + 1) / 2)
                       : C::PAIR_AXIS ? int64_t(a.tiles_m) * ((a.tiles_r + 1) / 2)
                                      : int64_t((a.tiles_m + C::CLUSTER - 1) / C::CLUSTER) *
                                            a.tiles_r;
  return i8_launch<C>(linear_solve_kernel<P, CL>, units, sms, s, tx, tw, tout, a, twh);
}

// Per-p entry of the split grid (kernels_lin_*.cu).
struct LinOps {
  int kt = 0, p8 = 0, rb = 0;
  // [0]: one CTA per tile; [1]: CTA pairs sharing (multicasting) the B tile;
  // [2]: CTA pairs on two B tiles sharing (multicasting) the SNP tile;
  // [3]: CTA pairs running one cta_group::2 MMA (32-row W tiles; else null)
  // [4]: 2 x 2 clusters multicasting halves of both operands
  cudaError_t (*launch[5])(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                           const LinArgs&, int, cudaStream_t, const CUtensorMap&) = {
      nullptr, nullptr, nullptr, nullptr, nullptr};
  // slice slots per TMA box (pairs / 2 x 2: the even rank's; the odd rank's
  // box holds the rest, 3 or 4 slots; pair MMA: + a half-slot box)
  int b_slices_box[5] = {I8_SEVEN_SLOTS ? 7 : 8, 4, I8_SEVEN_SLOTS ? 7 : 8, 3, 4};
  int a_box_rows[5] = {128, 128, 64, 128, 64};  // SNP rows per TMA box of the A tile
  int row = 0;           // doubles per TMA box row (LinCfg::BW)
  int cells = 0;         // traits per epilogue warp and tile (LinCfg::CELLS)
  int stream_rows = 0;   // rows (cells) of a stream-layout result box
  bool stream_tma = false;  // stream-layout results by TMA boxes {32p, cells}
  bool tma_row = false;  // results leave by unswizzled TMA boxes {row, 32}
  bool stream_stg = false;  // stream-layout results by direct 256-bit stores
  bool nostage = false;  // direct stores in any layout
  bool sbr_tma = false;  // tmap_out = the S_BR map
};

template <int P>
LinOps make_lin_ops() {
  LinOps o;
  o.kt = LinCfg<P>::KT;
  o.p8 = LinCfg<P>::P8;
  o.rb = LinCfg<P>::RB;
  o.launch[0] = &launch_linear_solve<P, 1>;
  o.launch[1] = &launch_linear_solve<P, 2>;
  o.launch[2] = &launch_linear_solve<P, 3>;
  if constexpr (LinCfg<P>::RB == 32) o.launch[3] = &launch_linear_solve<P, 4>;
  o.launch[4] = &launch_linear_solve<P, 5>;
  o.row = LinCfg<P>::BW;
  o.cells = LinCfg<P>::CELLS;
  o.stream_rows = LinCfg<P>::STREAM_HALF ? LinCfg<P>::GROUP : LinCfg<P>::CELLS;
  o.stream_tma = LinCfg<P>::STREAM_TMA;
  o.tma_row = LinCfg<P>::TMA_ROW;
  o.stream_stg = LinCfg<P>::STREAM_STG;
  o.nostage = LinCfg<P>::NOSTAGE;
  o.sbr_tma = LinCfg<P>::SBR_TMA;
  return o;
}

bool lin_ops_for_a(int64_t p, LinOps* out);  // p 1..16
bool lin_ops_for_b(int64_t p, LinOps* out);  // p 17..32
inline bool lin_ops_for(int64_t p, LinOps* out) {
  return lin_ops_for_a(p, out) || lin_ops_for_b(p, out);
}

}  // namespace gwg
