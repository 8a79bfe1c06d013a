// rotate_i8.cuh — exact-integer rotation of genotype-coded SNP slabs on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators).
//
// X' = Z^T X_R where X_R holds integer genotype codes (BASELINE.json: {0,1,2}).
// Each eigenvector z_r (column r of Z) is scaled by a power of two sigma_r
// (|z_r / sigma_r| <= 1/2), rounded to N_r = rint(2^55 z_r / sigma_r) and
// written as seven signed 8-bit base-256 digits (slice_basis_kernel),
//     z_r / sigma_r = 2^-55 sum_{s<7} d_{s,r} 256^(6-s) + O(2^-56),  |d| <= 128,
// so  X'[r, i] = sigma_r 2^-55 sum_s 256^(6-s) (d_{s,r} . x_i)  where every
// inner product is an EXACT int32 dot product of int8 vectors (|d x| <=
// 128*127, so exact for n < 132,000).  The seven partial results are combined
// exactly in int64 and converted with a single rounding, so X' is the
// correctly rounded value of sigma_r (55-bit expansion of z_r) . x_i — below a
// DGEMM's error — and each column depends only on (Z, x_i): bitwise identical
// for any slab width, like rotate_kernel.  The DMMA rotation
// (rotate_kernel.cuh) remains the general path for real-valued SNP data.
//
// GEMM view per CTA tile: M = 128 SNPs (A = X int8, K-major), N = 224 =
// 7 slices x 32 eigen-rows (B = slices in 8 smem slots, K-major), K = samples,
// int32 D in TMEM.  Warp roles: warp 0 = TMA producer (SWIZZLE_128B boxes,
// 4-stage mbarrier ring), warp 1 = MMA issuer (one thread, 4 x tcgen05.mma
// M128 N224 K32 per stage) and TMEM owner (2 x 224 columns: double-buffered
// accumulators), warps 4-11 = epilogue (tcgen05.ld 32x32b, exact int64
// recombination, X' and/or X'.X' tiles out through 128B-swizzled staging +
// TMA stores).
#pragma once

#include "i8_core.cuh"

namespace gwg {

struct I8Args {
  const double* scale;  // sigma_r per eigen-row (n)
  int32_t has_d;        // write X' through tmap_d
  int32_t has_d2;       // write X'.X' through tmap_d2
  int32_t n;            // eigen-rows (B columns): n for Z, t*p for W
  int32_t cols;
  int32_t tiles_m;      // ceil(cols / 128)
  int32_t tiles_r;      // ceil(n / 32)
  int32_t kstages;      // kp / 128
  int32_t b_resident;   // sliced operand fits L2: keep it resident
  const unsigned long long* gate = nullptr;  // GWG_SNP_AUTO path gate (gate_closed)
  int32_t gate_codes = 0;
  int32_t raster = 0;   // I8Sched raster (1: eigen-row tiles fastest)
};

// ---- the rotation kernel -------------------------------------------------------

// CL: 1 single CTAs, 2 CTA pairs multicasting B, 4 CTA pairs running one
// cta_group::2 MMA with half of B each (30 KB stages, 6 deep)
#ifndef ROT_WS  // producer and MMA loops warp-collective (I8Tile WS; measured slower here)
#define ROT_WS 0
#endif
template <int CL>
using RotI8Cfg = std::conditional_t<CL == 4, I8Tile<32, 6, 1, 8, 2, 0, 0, true, ROT_WS != 0>,
                                    I8Tile<32, 4, 1, 8, CL, 0, 0, false, ROT_WS != 0>>;

template <int CL>
__global__ void __launch_bounds__(RotI8Cfg<CL>::THREADS, 1)
    rotate_i8_kernel(const __grid_constant__ CUtensorMap tmap_x,
                     const __grid_constant__ CUtensorMap tmap_z,
                     const __grid_constant__ CUtensorMap tmap_d,
                     const __grid_constant__ CUtensorMap tmap_d2, const I8Args a,
                     const __grid_constant__ CUtensorMap tmap_zh) {
  if (gate_closed(a.gate, a.gate_codes)) return;
  using C = RotI8Cfg<CL>;
  static_assert(C::ACC_BUFS == 2, "epilogue alternates two accumulator buffers");
  extern __shared__ __align__(1024) unsigned char smem_i8[];
  const I8Smem<C> sm(smem_i8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const I8Sched<C> sch(a.tiles_m, a.tiles_r, a.raster);
  const int my_tiles = sch.my_tiles;
  const uint32_t tmem_base = i8_setup<C>(sm, warp);

  if (warp == 0) {
    if (C::WS || lane == 0)
      i8_produce<C>(sm, &tmap_x, &tmap_z, sch, a.kstages, a.b_resident != 0, &tmap_zh);
  } else if (warp == 1) {
    if (C::WS || lane == 0) i8_mma<C>(sm, tmem_base, my_tiles, a.kstages);
  } else if (warp >= 4) {
    // ---- epilogue: warp w reads TMEM lanes 32*(w%4).. (its SNP quarter) and
    // columns h*16..h*16+15 of every slice; exact int64 recombination (see
    // i8_recombine), rows to a 128B-swizzled staging tile, out by TMA store
    // (coalesced, clipped at the edges).
    const int ew = warp - 4;
    const int qd = warp & 3;
    const int h = ew >> 2;
    unsigned char* stg = sm.staging + ew * C::OUT_BYTES;
    for (int lt = 0; lt < my_tiles; ++lt) {
      const int buf = lt & 1;
      int tm, tr;
      sch.coords(lt, tm, tr);
      const int r0 = tr * C::RB + h * C::OUT_Q;
      double x[C::OUT_Q];
      mbar_wait(&sm.acc_full[buf], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + (uint32_t(qd * 32) << 16) + uint32_t(buf * C::BN + h * C::OUT_Q);
#pragma unroll
      for (int c = 0; c < C::OUT_Q / 8; ++c) {
        double sc[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int row = r0 + c * 8 + r;
          sc[r] = row < a.n ? __ldg(a.scale + row) : 0.0;  // sigma 2^-55
        }
        int32_t v[C::SLICES][8];
#pragma unroll
        for (int sl = 0; sl < C::SLICES; ++sl) tmem_ld8(taddr + uint32_t(sl * C::RB + c * 8), v[sl]);
        tmem_ld_wait();
#pragma unroll
        for (int r = 0; r < 8; ++r)
          x[c * 8 + r] = i8_recombine(v[0][r], v[1][r], v[2][r], v[3][r], v[4][r], v[5][r],
                                      v[6][r], sc[r]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) i8_acc_release<C>(sm, buf);  // TMEM buffer free for the next tile
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        if (!(o == 0 ? a.has_d : a.has_d2)) continue;
        if (lane == 0) bulk_wait_read0();  // the previous store has left the staging tile
        __syncwarp();
#pragma unroll
        for (int ch = 0; ch < C::OUT_Q / 2; ++ch) {
          double2 w;
          w.x = o == 0 ? x[2 * ch] : x[2 * ch] * x[2 * ch];
          w.y = o == 0 ? x[2 * ch + 1] : x[2 * ch + 1] * x[2 * ch + 1];
          *reinterpret_cast<double2*>(stg + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tma_store_2d(o == 0 ? &tmap_d : &tmap_d2, stg, r0, tm * C::BM + qd * 32);
      }
    }
    if (lane == 0) bulk_wait0();
  }
  i8_teardown<C>(tmem_base, warp);
}

// ---- slab / basis preparation ------------------------------------------------------

// X (n x cols, ld lds, f64 genotype codes) -> int8 [col][kp] with zero padding;
// flags (*bad = 0) any value that is not an integer in [-127, 127].  HBM-bound
// (8 bytes in, 1 out per code).  A block takes SNP_I8_ITEMS columns at a time
// and each thread one 16-byte code pair of every one of them (lds is even:
// 16-byte aligned columns), all loads issued before any conversion: bytes in
// flight without a full SM, so a grid of a few blocks per SM saturates HBM and
// leaves room on every SM for the trait-side kernels that run concurrently
// (split_build_ahead).
#ifndef SNP_I8_ITEMS
#define SNP_I8_ITEMS 4
#endif
__global__ void __launch_bounds__(256) snp_to_i8_kernel(const double* __restrict__ x, int64_t lds,
                                                        int32_t n, int32_t cols, int32_t kp,
                                                        int8_t* __restrict__ out,
                                                        unsigned long long* __restrict__ bad) {
  constexpr int U = SNP_I8_ITEMS;
  bool ok = true;
  const int pairs = kp >> 1;
  for (int c0 = blockIdx.x * U; c0 < cols; c0 += gridDim.x * U) {
    for (int k2 = threadIdx.x; k2 < pairs; k2 += blockDim.x) {
      const int k = 2 * k2;
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = make_double2(0.0, 0.0);
        const double* col = x + int64_t(c0 + u) * lds;
        if (c0 + u < cols) {
          if (k + 1 < n)
            v[u] = __ldcs(reinterpret_cast<const double2*>(col + k));
          else if (k < n)
            v[u].x = col[k];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + u >= cols) continue;
        const bool good = (v[u].x == rint(v[u].x)) & (fabs(v[u].x) <= 127.0) &
                          (v[u].y == rint(v[u].y)) & (fabs(v[u].y) <= 127.0);
        ok &= good;
        reinterpret_cast<uint16_t*>(out + int64_t(c0 + u) * kp)[k2] =
            good ? uint16_t((uint32_t(int(v[u].x)) & 0xffu) |
                            ((uint32_t(int(v[u].y)) & 0xffu) << 8))
                 : uint16_t(0);
      }
    }
  }
  if (!ok) *bad = 0;  // error words are reset to all ones
}

// Z (n x ncols, ld ldz) -> slices [s][r][kp] int8 and scale[r] = sigma_r 2^-55 (the
// factor that turns the recombined integer into the value, exact): one
// block per column r (an eigenvector of Z, or a column of W for the split grid).
// v = z / sigma (exact, |v| <= 1/2), N = rint(v 2^55) (|N| <= 2^54), written
// in balanced base 256: N = sum_s d_s 256^(6-s) with d_6..d_1 in [-128, 127]
// and |d_0| <= 65, so every digit is an int8 and the column is sigma 2^-55 N
// (relative to sigma, within 2^-56 of z / sigma).
__global__ void slice_basis_kernel(const double* __restrict__ z, int64_t ldz, int32_t n,
                                   int32_t ncols, int32_t kp, int8_t* __restrict__ slices,
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
    scale[r] = red[0] * 0x1p-55;
  }
  __syncthreads();
  const double inv = 1.0 / red[0];  // exact: power of two
  const int64_t plane = int64_t(ncols) * kp;
  for (int k = threadIdx.x; k < kp; k += blockDim.x) {
    const double v = k < n ? col[k] * inv : 0.0;  // exact scaling
    long long q = llrint(v * 0x1p55);             // exact scaling, one rounding
#pragma unroll
    for (int s = I8Cfg::SLICES - 1; s >= 0; --s) {
      const long long d = ((q + 128) & 255) - 128;
      slices[s * plane + int64_t(r) * kp + k] = int8_t(d);
      q = (q - d) >> 8;  // exact: q - d is a multiple of 256
    }
  }
}

}  // namespace gwg
