// engine.cu — host engine + C ABI (include/gwgrid_cuda.h) of the B200 GLS grid.
//
// Reference seams replaced here (proj/include/gwgrid/grid.hpp):
//   precompute_grid / GridPrecompute        -> gwg_set_spectrum + gwg_set_covariates
//   transform_trait_slab + build_trait_contexts + load_pass -> gwg_set_traits
//   transform_snp_slab + compute_tile        -> gwg_solve_snp_slab
//   preloop_stream_transform + run_grid (CT, double-buffered pipeline_run,
//   pipeline.hpp:78-137)                     -> gwg_run_grid
// Every kernel on the path is this library's own sm_100a code: the
// deterministic FP64-DMMA rotation (rotate_kernel.cuh) and its exact int8
// tcgen05 counterpart for genotype slabs (rotate_i8.cuh), the per-trait
// context kernel (trait_prep.cuh), the fused FP64 grid kernel
// (grid_kernel.cuh) and the genotype split grid (grid_split.cuh: S_BR on DMMA;
// linear_solve.cuh: exact int8 linear terms fused with the Cholesky solve).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gwgrid_cuda.h"
#include "split_prep.cuh"
#include "engine_internal.cuh"
#include "rotate_i8.cuh"
#include "rotate_kernel.cuh"
#include "slab_kernels.cuh"

#ifndef LIN_RASTER
#define LIN_RASTER 0  // trait tiles fastest: measured 2.49-2.54 vs 2.45-2.46 ms at c1 (off)
#endif
#ifndef GWG_B_RESIDENT_MB  // sliced operands up to this size are loaded evict_last
#define GWG_B_RESIDENT_MB 48
#endif
#ifndef GWG_PERSIST_L2_MB  // L2 set-aside for persisting (evict_last) lines, MB (0 = leave)
#define GWG_PERSIST_L2_MB 0
#endif
#ifndef SNP_I8_BLOCKS  // blocks per SM of the code conversion
#define SNP_I8_BLOCKS 8
#endif
#ifndef SNP_I8_BLOCKS_BESIDE  // the same with the trait side running beside it
#define SNP_I8_BLOCKS_BESIDE 8    // 2 (+ GWG_SMEM_CARVEOUT): measured neutral, off (below)
#endif
#ifndef GWG_COV_STREAM  // W's covariate columns on a helper stream beside the trait column
#define GWG_COV_STREAM 0  // measured neutral at c1 (the rotation holds the SMs the covariate GEMMs need)
#endif
#ifndef GWG_TRAITS_ON_SIDE  // gwg_set_traits' device work on the side stream (split path)
#define GWG_TRAITS_ON_SIDE 1
#endif
#ifndef GWG_SIDE_PRIORITY
#define GWG_SIDE_PRIORITY 1
#endif
// stream layout by direct 256-bit stores (p % 4 == 0) instead of TMA boxes
#ifndef LIN_STREAM_STG
#define LIN_STREAM_STG 0
#endif
#ifndef LIN_STREAM_TMA
#define LIN_STREAM_TMA 1
#endif
#ifndef ROT_RASTER
#define ROT_RASTER 0  // eigen-row tiles fastest: neutral at c1 (off)
#endif

namespace gwg_host {

using gwg::kBK;
using gwg::KernelOps;

int set_status(gwg_status* st, int code, int64_t snp, int64_t trait, const char* fmt, ...) {
  if (st) {
    st->code = code;
    st->snp_index = snp;
    st->trait_index = trait;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

void clear_status(gwg_status* st) {
  if (st) {
    st->code = GWG_OK;
    st->snp_index = -1;
    st->trait_index = -1;
    st->msg[0] = 0;
  }
}

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int check_engine(gwg_engine* e, gwg_status* st, bool join) {
  if (!e) return set_status(st, GWG_DIMENSION, -1, -1, "null engine");
  cudaError_t err = cudaSetDevice(e->device);
  if (err != cudaSuccess)
    return set_status(st, GWG_CUDA, -1, -1, "cudaSetDevice: %s", cudaGetErrorString(err));
  if (join) GWG_CUDA_TRY(join_side(e));
  return GWG_OK;
}

// The compute stream waits for the trait-side work queued on the side stream.
cudaError_t join_side(gwg_engine* e) {
  if (!e->side_pending) return cudaSuccess;
  e->side_pending = false;
  cudaError_t err = cudaEventRecord(e->ev_join, e->side);
  if (err == cudaSuccess) err = cudaStreamWaitEvent(e->comp, e->ev_join, 0);
  return err;
}

int upload(gwg_engine* e, DevBuf& dst, const double* src, size_t count, int where,
           gwg_status* st) {
  GWG_CUDA_TRY(dst.ensure(std::max<size_t>(count, 1) * sizeof(double)));
  if (count == 0) return GWG_OK;
  // device operands may live on another GPU (the group's peer broadcast):
  // cudaMemcpyDefault lets UVA pick the route
  GWG_CUDA_TRY(cudaMemcpyAsync(dst.ptr, src, count * sizeof(double),
                               where == GWG_DEVICE ? cudaMemcpyDefault : cudaMemcpyHostToDevice,
                               e->comp));
  if (where != GWG_DEVICE) e->counters.bytes_loaded += count * sizeof(double);
  return GWG_OK;
}

// Upload an n x cols column-major operand (leading dimension lds) into dst
// with leading dimension np (the TMA-aligned layout every kernel reads).
int upload_cols(gwg_engine* e, DevBuf& dst, const double* src, int64_t lds, int64_t cols,
                int where, cudaStream_t s, gwg_status* st, int64_t ldd) {
  if (ldd == 0) ldd = e->np;
  GWG_CUDA_TRY(dst.ensure(size_t(ldd) * std::max<int64_t>(cols, 1) * sizeof(double)));
  if (cols == 0) return GWG_OK;
  const cudaMemcpyKind kind = where == GWG_DEVICE ? cudaMemcpyDefault : cudaMemcpyHostToDevice;
  if (lds == e->n && ldd == e->n) {
    GWG_CUDA_TRY(cudaMemcpyAsync(dst.ptr, src, size_t(e->n) * cols * sizeof(double), kind, s));
  } else {
    GWG_CUDA_TRY(cudaMemcpy2DAsync(dst.ptr, ldd * sizeof(double), src, lds * sizeof(double),
                                   e->n * sizeof(double), cols, kind, s));
  }
  if (where != GWG_DEVICE) e->counters.bytes_loaded += uint64_t(e->n) * cols * 8;
  return GWG_OK;
}

int encode_kmajor(CUtensorMap* map, const double* base, int64_t n, int64_t rows, int64_t ld,
                  int box_rows, gwg_status* st) {
  auto encode = get_encode();
  if (!encode) return set_status(st, GWG_CUDA, -1, -1, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t gdim[2] = {cuuint64_t(n), cuuint64_t(rows)};
  const cuuint64_t gstride[1] = {cuuint64_t(ld) * sizeof(double)};
  const cuuint32_t box[2] = {8, cuuint32_t(box_rows)};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim,
                      gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_status(st, GWG_CUDA, -1, -1, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return GWG_OK;
}

// Leading dimension for raw operands: n itself when TMA can address it
// (row pitch a multiple of 16 bytes), so host slabs move with one flat copy.
int64_t raw_ld(const gwg_engine* e) { return (e->n % 2 == 0) ? e->n : e->np; }

// dst (n x cols, ld np) = Z^T src (n x cols, ld lds) with the deterministic
// DMMA rotation kernel (rotate_kernel.cuh).
int rotate(gwg_engine* e, const double* src, int64_t cols, double* dst, gwg_status* st,
           int64_t lds, double* dst_sq, const double* basis, int64_t ldd) {
  if (cols <= 0) return GWG_OK;
  NvtxRange nvtx_("rotate");
  if (lds == 0) lds = e->np;
  if (ldd == 0) ldd = e->np;
  CUtensorMap tz, tx;
  if (!basis) basis = e->basis.d();
  if (int rc = encode_kmajor(&tz, basis, e->n, e->n, e->np, gwg::RotCfg::BM, st)) return rc;
  if (int rc = encode_kmajor(&tx, src, e->n, cols, lds, gwg::RotCfg::BN, st)) return rc;
  gwg::RotArgs a;
  a.dst = dst;
  a.dst_sq = dst_sq;
  a.ldd = ldd;
  a.n = int32_t(e->n);
  a.cols = int32_t(cols);
  a.tiles_m = int32_t(ceil_div(e->n, gwg::RotCfg::BM));
  a.tiles_n = int32_t(ceil_div(cols, gwg::RotCfg::BN));
  a.kchunks = int32_t(e->np / gwg::RotCfg::BK);
  a.gate = gate_word(e);
  a.gate_codes = e->gate_want;
  const int64_t tiles = int64_t(a.tiles_m) * a.tiles_n;
  GWG_CUDA_TRY(gwg::launch_rotate(tz, tx, a, int(std::min<int64_t>(tiles, e->sms)), e->comp));
  e->counters.kernel_launches += 1;
  e->counters.preloop_flops += 2ull * uint64_t(e->n) * uint64_t(e->n) * uint64_t(cols);
  return GWG_OK;
}

int read_errors(gwg_engine* e, gwg_status* st, bool slab_checks) {
  GWG_CUDA_TRY(join_side(e));  // the trait word is written by the context build
  GWG_CUDA_TRY(cudaMemcpyAsync(e->err_host, e->err.ptr, 3 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, e->comp));
  GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));
  if (e->err_host[0] != ~0ull) {  // queued by gwg_set_traits, reported here
    const int64_t j = int64_t(e->err_host[0]);
    return set_status(st, GWG_NOT_POSITIVE_DEFINITE, -1, j,
                      "trait covariance is not positive definite in the rotated basis: a "
                      "weight entry is below the relative floor (trait %lld)",
                      (long long)j);
  }
  if (!slab_checks) return GWG_OK;
  if (e->i8_input && e->err_host[2] != ~0ull)
    return set_status(st, GWG_DIMENSION, -1, -1,
                      "int8 SNP slabs must hold genotype codes in [-127, 127] (found -128)");
  if (e->snp_coding == GWG_SNP_GENOTYPES && e->err_host[2] != ~0ull)
    return set_status(st, GWG_DIMENSION, -1, -1,
                      "SNP values are not integer genotype codes in [-127, 127] "
                      "(gwg_set_snp_coding(GENOTYPES)); use real-valued coding");
  return GWG_OK;
}

int reset_errors(gwg_engine* e, gwg_status* st) {
  GWG_CUDA_TRY(cudaMemsetAsync(static_cast<unsigned long long*>(e->err.ptr) + 1, 0xff,
                               2 * sizeof(unsigned long long), e->comp));
  return GWG_OK;
}

int begin_epoch(gwg_engine* e, gwg_status* st) {
  if (e->epoch_open) return GWG_OK;
  if (int rc = reset_errors(e, st)) return rc;
  e->epoch_open = true;
  return GWG_OK;
}

int end_epoch(gwg_engine* e, gwg_status* st) {
  const int rc = read_errors(e, st, true);  // synchronises the compute stream
  for (size_t k = e->timings_first; k < e->timings_used; ++k) {
    const auto& tm = e->timings[k];
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, tm.ev[0], tm.ev[1]) == cudaSuccess) e->counters.rotate_ms += ms;
    if (tm.joined && cudaEventElapsedTime(&ms, tm.ev[7], tm.ev[8]) == cudaSuccess)
      e->counters.rotate_ms -= ms;  // waiting for the trait side is not rotation
    if (cudaEventElapsedTime(&ms, tm.ev[2], tm.ev[3]) == cudaSuccess) e->counters.grid_kernel_ms += ms;
    if (tm.split) {
      if (cudaEventElapsedTime(&ms, tm.ev[4], tm.ev[5]) == cudaSuccess) e->counters.quad_ms += ms;
      if (cudaEventElapsedTime(&ms, tm.ev[5], tm.ev[6]) == cudaSuccess) e->counters.linear_ms += ms;
    }
  }
  cudaGetLastError();  // an event of a failed launch never recorded
  e->timings_used = e->timings_first = 0;
  e->epoch_open = false;
  if (rc) return rc;
  return raise_cell_error(e, st);
}

// The int8 kernels' default launch geometry: CTA pairs running one
// cta_group::2 MMA (half of the sliced operand per CTA, deeper operand rings)
// once a tile has at least 16 K stages; below that the B-multicast pairs.
// Measured (ms; B pairs -> pair MMA): rotation n = 1000 0.686 -> 0.745,
// n = 2000 1.104 -> 1.092, n = 4000 3.85 -> 3.64, n = 10,000 44.4 -> 41.1;
// linear_solve p = 4 n = 1000 2.40 -> 2.77, n = 2000 2.15 -> 2.10, n = 4000
// 4.02 -> 3.69, n = 6000 6.01 -> 5.21, n = 10,000 22.1 -> 18.3.
inline bool pair_mma_default(int64_t kp) { return kp / gwg::I8Cfg::BK >= 16; }

// 2-D uint8 map over a K-major int8 operand (kp x cols) and 3-D map over
// SLICES planes of (kp x ncols), both SWIZZLE_128B boxes for tcgen05.
int encode_i8(CUtensorMap* tx, const void* x, int64_t kp, int64_t cols, CUtensorMap* tb,
              const void* slices, int64_t ncols, int rb, int slices_box, gwg_status* st,
              int a_rows, CUtensorMap* tbh) {
  using gwg::I8Cfg;
  auto encode = get_encode();
  if (!encode) return set_status(st, GWG_CUDA, -1, -1, "cuTensorMapEncodeTiled unavailable");
  {
    const cuuint64_t gdim[2] = {cuuint64_t(kp), cuuint64_t(cols)};
    const cuuint64_t gstride[1] = {cuuint64_t(kp)};
    const cuuint32_t box[2] = {I8Cfg::BK, cuuint32_t(a_rows)};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(x), gdim, gstride,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return set_status(st, GWG_CUDA, -1, -1, "tensor map (int8 SNP slab) failed (%d)", int(r));
  }
  {
    const cuuint64_t gdim[3] = {cuuint64_t(kp), cuuint64_t(ncols), cuuint64_t(I8Cfg::SLICES)};
    const cuuint64_t gstride[2] = {cuuint64_t(kp), cuuint64_t(ncols) * kp};
    const cuuint32_t box[3] = {I8Cfg::BK, cuuint32_t(rb), cuuint32_t(slices_box)};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(slices), gdim,
                        gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return set_status(st, GWG_CUDA, -1, -1, "tensor map (int8 slices) failed (%d)", int(r));
    // the half-slot box of the pair MMA (I8Tile MMA2): rb/2 rows of one slice;
    // for CTA pairs / 2 x 2 clusters the odd rank's box: the slots after the
    // even rank's 4 (3 real slices with I8_SEVEN_SLOTS); otherwise tb itself
    const cuuint32_t hbox[3] = {I8Cfg::BK, cuuint32_t(rb / 2), 1};
    const cuuint32_t obox[3] = {I8Cfg::BK, cuuint32_t(rb),
                                cuuint32_t(I8_SEVEN_SLOTS ? I8Cfg::SLICES - 4 : 4)};
    r = tbh == nullptr ? CUDA_SUCCESS
        : slices_box == 3 || slices_box == 4
            ? encode(tbh, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(slices), gdim,
                     gstride, slices_box == 3 ? hbox : obox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
            : (*tbh = *tb, CUDA_SUCCESS);
    if (r != CUDA_SUCCESS)
      return set_status(st, GWG_CUDA, -1, -1, "tensor map (int8 half slices) failed (%d)", int(r));
  }
  return GWG_OK;
}

// rotate_i8_kernel over `cols` int8 SNP columns against the sliced columns
// (scale, ncols): dst[i * ldd + r] (and dst_sq) for r < ncols, either may be
// null.  Outputs leave through TMA stores: ldd even, 16-byte aligned bases.
int launch_i8(gwg_engine* e, const void* xi8, const void* slices, int64_t cols, int64_t ncols,
              const double* scale, double* dst, double* dst_sq, int64_t ldd, gwg_status* st) {
  using gwg::I8Cfg;
  auto encode = get_encode();
  if (!encode) return set_status(st, GWG_CUDA, -1, -1, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap td[2];
  double* outs[2] = {dst, dst_sq};
  for (int o = 0; o < 2; ++o) {
    double* base = outs[o] ? outs[o] : (dst ? dst : dst_sq);
    const cuuint64_t gdim[2] = {cuuint64_t(ncols), cuuint64_t(cols)};
    const cuuint64_t gstride[1] = {cuuint64_t(ldd) * 8};
    const cuuint32_t box[2] = {I8Cfg::OUT_Q, 32};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&td[o], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, gdim, gstride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return set_status(st, GWG_CUDA, -1, -1, "tensor map (int8 rotation output) failed (%d)",
                        int(r));
  }
  const int64_t kp = round_up(e->n, I8Cfg::BK);
  gwg::I8Args a;
  a.scale = scale;
  a.has_d = dst != nullptr;
  a.has_d2 = dst_sq != nullptr;
  a.n = int32_t(ncols);
  a.cols = int32_t(cols);
  a.tiles_m = int32_t(ceil_div(cols, I8Cfg::BM));
  a.tiles_r = int32_t(ceil_div(ncols, I8Cfg::RB));
  a.kstages = int32_t(kp / I8Cfg::BK);
  a.b_resident = size_t(I8Cfg::SLICES) * ncols * kp <= (size_t(GWG_B_RESIDENT_MB) << 20);
  a.gate = gate_word(e);
  a.gate_codes = e->gate_want;
  a.raster = (ROT_RASTER == 2 || (ROT_RASTER == 1 && a.b_resident)) ? 1 : 0;
  // CTA pairs multicasting the B (Z-slice) tile: halves its L2 -> SMEM
  // traffic (the rotation runs at ~77% of L2 throughput with single CTAs);
  // measured at n = 10,000: 69.2 -> 49.0 ms, at n = 1000: 0.704 -> 0.692 ms
  // GWG_OPT_I8_CLUSTER = 4: CTA pairs running one cta_group::2 MMA with half
  // of the Z-slice tile each — the default from 16 K stages (n > 1920) on
  // (pair_mma_default)
  const int cl = e->i8_cluster ? (e->i8_cluster == 3 || e->i8_cluster == 5 ? 2 : e->i8_cluster)
                               : pair_mma_default(kp) ? 4 : 2;
  CUtensorMap tx, tb, tbh;
  if (int rc = encode_i8(&tx, xi8, kp, cols, &tb, slices, ncols, I8Cfg::RB,
                         cl == 4 ? 3 : cl == 1 ? (I8_SEVEN_SLOTS ? 7 : 8) : 4, st, I8Cfg::BM,
                         &tbh))
    return rc;
  const int pair = cl >= 2 ? 2 : 1;
  const int64_t units = int64_t((a.tiles_m + pair - 1) / pair) * a.tiles_r;
  if (cl == 4)
    GWG_CUDA_TRY(gwg::i8_launch<gwg::RotI8Cfg<4>>(gwg::rotate_i8_kernel<4>, units, e->sms,
                                                  e->comp, tx, tb, td[0], td[1], a, tbh));
  else if (cl == 2)
    GWG_CUDA_TRY(gwg::i8_launch<gwg::RotI8Cfg<2>>(gwg::rotate_i8_kernel<2>, units, e->sms,
                                                  e->comp, tx, tb, td[0], td[1], a, tbh));
  else
    GWG_CUDA_TRY(gwg::i8_launch<gwg::RotI8Cfg<1>>(gwg::rotate_i8_kernel<1>, units, e->sms,
                                                  e->comp, tx, tb, td[0], td[1], a, tbh));
  e->counters.kernel_launches += 1;
  return GWG_OK;
}

int rotate_snps(gwg_engine* e, const double* src, int64_t lds, int64_t cols, gwg_status* st) {
  e->slab_i8 = false;
  e->slab_auto = false;
  const bool i8_ok = e->n < kMaxGenotypeN;
  if (e->snp_coding == GWG_SNP_REAL || (e->snp_coding == GWG_SNP_AUTO && !i8_ok))
    return rotate(e, src, cols, e->rot.d(), st, lds, e->rot_sq.d());
  if (cols <= 0) return GWG_OK;
  const bool autom = e->snp_coding == GWG_SNP_AUTO;
  if (autom)  // this slab's verdict alone decides its path
    GWG_CUDA_TRY(cudaMemsetAsync(static_cast<unsigned long long*>(e->err.ptr) + 2, 0xff,
                                 sizeof(unsigned long long), e->comp));
  NvtxRange nvtx_("rotate_i8");
  using gwg::I8Cfg;
  const int64_t n = e->n, kp = round_up(n, I8Cfg::BK);
  if (!e->slices_valid) {
    GWG_CUDA_TRY(e->zslices.ensure(size_t(I8Cfg::SLICES) * n * kp));
    GWG_CUDA_TRY(e->zscale.ensure(size_t(n) * sizeof(double)));
    gwg::prefer_max_smem(gwg::slice_basis_kernel);
    gwg::slice_basis_kernel<<<int(n), 256, 0, e->comp>>>(
        e->basis.d(), e->np, int32_t(n), int32_t(n), int32_t(kp),
        static_cast<int8_t*>(e->zslices.ptr), e->zscale.d());
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    e->slices_valid = true;
  }
  GWG_CUDA_TRY(e->xi8.ensure(size_t(cols) * kp));
  {
    // HBM-bound, all blocks resident.  Measured and not kept: two blocks per
    // SM plus the max-shared carveout (SNP_I8_BLOCKS_BESIDE = 2,
    // GWG_SMEM_CARVEOUT = 1) whenever the trait side runs beside it — its
    // 200 KB-CTA rotations then co-reside from the start instead of waiting
    // for the conversion to drain (c1 "other" 0.31 -> 0.19 ms), but the
    // conversion slows by the same 0.12 ms (step 4.23-4.27 vs 4.23-4.24 ms).
    const bool beside = e->side_pending || (e->fork_pending && !e->split_valid);
    const int per_sm = beside ? SNP_I8_BLOCKS_BESIDE : SNP_I8_BLOCKS;
    const int blocks = int(std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(cols, SNP_I8_ITEMS), int64_t(e->sms) * per_sm)));
    if (GWG_SMEM_CARVEOUT) {
      cudaFuncSetAttribute(reinterpret_cast<const void*>(gwg::snp_to_i8_kernel),
                           cudaFuncAttributePreferredSharedMemoryCarveout,
                           beside ? int(cudaSharedmemCarveoutMaxShared)
                                  : int(cudaSharedmemCarveoutDefault));
      (void)cudaGetLastError();
    }
    gwg::snp_to_i8_kernel<<<blocks, 256, 0, e->comp>>>(
        src, lds, int32_t(n), int32_t(cols), int32_t(kp), static_cast<int8_t*>(e->xi8.ptr),
        static_cast<unsigned long long*>(e->err.ptr) + 2);
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
  }
  if (int rc = split_build_ahead(e, st)) return rc;
  // the split grid needs only X'.X' (its linear terms come from the codes)
  if (autom) e->gate_want = 1;
  int rc = launch_i8(e, e->xi8.ptr, e->zslices.ptr, cols, n, e->zscale.d(),
                     e->split ? nullptr : e->rot.d(), e->rot_sq.d(), e->np, st);
  if (autom && rc == GWG_OK) {  // the FP64 rotation for a slab with non-code values
    e->gate_want = 0;
    rc = rotate(e, src, cols, e->rot.d(), st, lds, e->rot_sq.d());
  }
  e->gate_want = -1;
  if (rc) return rc;
  e->counters.preloop_flops += 2ull * uint64_t(n) * uint64_t(n) * uint64_t(cols);
  e->slab_i8 = true;
  e->slab_auto = autom;
  return GWG_OK;
}

// int8 genotype slab (GWG_FORMAT_I8: n x cols codes, ld n) -> X'.X' (the
// genotype path) or, for GWG_SNP_REAL / n beyond the exact-int8 bound, FP64
// codes -> the DMMA rotation.  Codes are codes: no per-slab verdict gates
// the launches; a -128 is an error (read_errors).
int rotate_snps_i8(gwg_engine* e, const int8_t* src, int64_t cols, gwg_status* st) {
  e->slab_i8 = false;
  e->slab_auto = false;
  if (cols <= 0) return GWG_OK;
  using gwg::I8Cfg;
  const int64_t n = e->n, kp = round_up(n, I8Cfg::BK);
  const int blocks = int(std::min<int64_t>(cols, int64_t(e->sms) * 16));
  if (e->snp_coding == GWG_SNP_REAL || n >= kMaxGenotypeN) {
    GWG_CUDA_TRY(e->stage.ensure(size_t(raw_ld(e)) * cols * sizeof(double)));
    gwg::i8_unpack_kernel<<<blocks, 256, 0, e->comp>>>(src, int32_t(n), int32_t(cols),
                                                       e->stage.d(), raw_ld(e));
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    const int saved = e->snp_coding;
    e->snp_coding = GWG_SNP_REAL;
    const int rc = rotate_snps(e, e->stage.d(), raw_ld(e), cols, st);
    e->snp_coding = saved;
    return rc;
  }
  NvtxRange nvtx_("rotate_i8");
  if (!e->slices_valid) {
    GWG_CUDA_TRY(e->zslices.ensure(size_t(I8Cfg::SLICES) * n * kp));
    GWG_CUDA_TRY(e->zscale.ensure(size_t(n) * sizeof(double)));
    gwg::prefer_max_smem(gwg::slice_basis_kernel);
    gwg::slice_basis_kernel<<<int(n), 256, 0, e->comp>>>(
        e->basis.d(), e->np, int32_t(n), int32_t(n), int32_t(kp),
        static_cast<int8_t*>(e->zslices.ptr), e->zscale.d());
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    e->slices_valid = true;
  }
  GWG_CUDA_TRY(e->xi8.ensure(size_t(cols) * kp));
  gwg::i8_pack_kernel<<<blocks, 256, 0, e->comp>>>(
      src, int32_t(n), int32_t(cols), int32_t(kp), static_cast<int8_t*>(e->xi8.ptr),
      static_cast<unsigned long long*>(e->err.ptr) + 2);
  GWG_CUDA_TRY(cudaGetLastError());
  e->counters.kernel_launches += 1;
  if (int rc = split_build_ahead(e, st)) return rc;
  if (int rc = launch_i8(e, e->xi8.ptr, e->zslices.ptr, cols, n, e->zscale.d(),
                         e->split ? nullptr : e->rot.d(), e->rot_sq.d(), e->np, st))
    return rc;
  e->counters.preloop_flops += 2ull * uint64_t(n) * uint64_t(n) * uint64_t(cols);
  e->slab_i8 = true;
  return GWG_OK;
}

int launch_checksum(gwg_engine* e, const double* out, int64_t rows, int layout, int64_t i0,
                    gwg_status* st) {
  const bool numpy = layout == GWG_LAYOUT_NUMPY;
  const int64_t outer = numpy ? rows : e->t, inner = numpy ? e->t : rows;
  const int blocks = int(std::min<int64_t>(outer, int64_t(e->sms) * 8));
  gwg::checksum_kernel<<<blocks, 256, 0, e->comp>>>(out, outer, inner, int32_t(e->p),
                                                    numpy ? 1 : 0, i0,
                                                    static_cast<unsigned long long*>(e->csum.ptr));
  GWG_CUDA_TRY(cudaGetLastError());
  e->counters.kernel_launches += 1;
  e->csum_cells += uint64_t(rows) * uint64_t(e->t);
  return GWG_OK;
}

bool rotated_x_unused(const gwg_engine* e) {
  if (!e->split) return false;
  if (e->i8_input) return e->snp_coding != GWG_SNP_REAL && e->n < kMaxGenotypeN;
  return e->snp_coding == GWG_SNP_GENOTYPES;
}

void invalidate_derived(gwg_engine* e, bool spectrum) {
  e->split_valid = false;
  e->expsum_valid = false;
  if (spectrum) {
    e->slices_valid = false;
    e->basis_t_valid = false;
  }
}

// min / max of the eigenvalues, once per spectrum (expsum_range_kernel with
// no traits, one round trip): the exponential sum's range needs them.
int spectrum_range(gwg_engine* e, gwg_status* st) {
  GWG_CUDA_TRY(e->exps.ensure(size_t(8 + 2 * 512) * sizeof(double)));
  double* dx = e->exps.d();
  gwg::prefer_max_smem(gwg::expsum_range_kernel);
  gwg::expsum_range_kernel<<<1, 256, 0, e->comp>>>(e->lambda.d(), e->n, nullptr, nullptr, 0,
                                                    dx);
  GWG_CUDA_TRY(cudaGetLastError());
  e->counters.kernel_launches += 1;
  double rg[6];
  GWG_CUDA_TRY(cudaMemcpyAsync(rg, dx, sizeof(rg), cudaMemcpyDeviceToHost, e->comp));
  GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));
  e->lam_lo = rg[0];
  e->lam_hi = rg[1];
  e->lam_bad = rg[5] != 0.0;
  e->ex_hi = -1.0;  // nodes must be redesigned
  return GWG_OK;
}

// E and F of the low-rank S_BR (expsum.cpp) for the current traits, or
// sbr_terms = 0 when D is outside the factorisation's range: some
// h lambda + 1 - h <= 0 (the trait check reports those), non-finite scales,
// or x_max / x_min so wide that more than kMaxTerms terms would be needed.
constexpr int32_t kMaxTerms = 512;
int build_expsum(gwg_engine* e, gwg_status* st) {
  e->sbr_terms = 0;
  if (!e->lowrank) return GWG_OK;
  const int64_t n = e->n, np = e->np, t = e->t;
  GWG_CUDA_TRY(e->exps.ensure(size_t(8 + 2 * kMaxTerms) * sizeof(double)));
  double* dx = e->exps.d();
  double rg[6];
  if (e->traits_host_valid) {
    // the same reduction as expsum_range_kernel: the spectrum's range was
    // found with the spectrum, the traits' from the host copies
    rg[0] = e->lam_lo, rg[1] = e->lam_hi, rg[2] = INFINITY, rg[3] = -INFINITY, rg[4] = 0.0;
    bool bad = e->lam_bad;
    for (int64_t j = 0; j < t; ++j) {
      const double h = e->h2_host[j], s2 = e->s2_host[j];
      if (h != 0.0) {
        const double g = (1.0 - h) / h;
        rg[2] = std::fmin(rg[2], g);
        rg[3] = std::fmax(rg[3], g);
        rg[4] += 1.0;
        bad |= !std::isfinite(g) || !std::isfinite(1.0 / (s2 * h));
      } else {
        bad |= !std::isfinite(1.0 / s2);
      }
    }
    rg[5] = bad ? 1.0 : 0.0;
  } else if (e->range_pending) {  // queued by gwg_set_traits
    GWG_CUDA_TRY(cudaEventSynchronize(e->ev_range));
    std::copy(e->range_host, e->range_host + 6, rg);
  } else {  // device-resident inputs: one small reduction and a round trip
    gwg::prefer_max_smem(gwg::expsum_range_kernel);
    gwg::expsum_range_kernel<<<1, 256, 0, e->comp>>>(e->lambda.d(), n, e->h2.d(),
                                                      e->sigma2.d(), int32_t(t), dx);
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    GWG_CUDA_TRY(cudaMemcpyAsync(rg, dx, sizeof(rg), cudaMemcpyDeviceToHost, e->comp));
    GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));
  }
  if (rg[5] != 0.0) return GWG_OK;
  double x_min = 1.0, x_max = 1.0;  // all h = 0: only the constant term is used
  if (rg[4] > 0.0) {
    x_min = rg[0] + rg[2];
    x_max = rg[1] + rg[3];
  }
  // r: a whole number of S_BR column tiles (GEMM 1) and k-chunks (GEMM 2)
  const int32_t mult = std::lcm(e->sops.bt, e->sops.bk);
  int32_t r = 0;
  if (x_min == e->ex_lo && x_max == e->ex_hi && mult == e->ex_mult) {
    r = e->ex_r;  // same range as the nodes already on the device
  } else {
    if (gwg_exp_sum_design(x_min, x_max, mult, kMaxTerms, nullptr, nullptr, &r) != GWG_OK)
      return GWG_OK;
    std::vector<double> nodes(2 * size_t(r));
    gwg_exp_sum_design(x_min, x_max, mult, kMaxTerms, nodes.data(), nodes.data() + r, &r);
    GWG_CUDA_TRY(cudaMemcpyAsync(dx + 8, nodes.data(), nodes.size() * sizeof(double),
                                 cudaMemcpyHostToDevice, e->comp));
    GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));  // `nodes` is pageable and local
    e->ex_lo = x_min, e->ex_hi = x_max, e->ex_mult = mult, e->ex_r = r;
  }
  const int64_t bt = e->sops.bt;
  const int64_t t_pad = round_up(t, bt);
  // (+ slack: the split-K G GEMM may read up to 7 K-chunks past the last
  // trait tile's panel; they meet zero-filled SNP-side tiles, so they only
  // have to be finite: zeroed)
  {
    const size_t panel = size_t(r) * np * sizeof(double);
    const size_t slack = size_t(8) * e->sops.bk * e->sops.bt * sizeof(double);
    GWG_CUDA_TRY(e->epanel.ensure(panel + slack));
    GWG_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(e->epanel.ptr) + panel, 0, slack, e->comp));
  }
  GWG_CUDA_TRY(e->fpanel.ensure(size_t(t_pad) * r * sizeof(double)));
  if (t_pad != t)  // padded traits of the last tile contribute zeros
    GWG_CUDA_TRY(cudaMemsetAsync(e->fpanel.d() + size_t(t_pad - bt) * r, 0,
                                 size_t(bt) * r * sizeof(double), e->comp));
  gwg::ExpSumArgs a;
  a.n = n;
  a.np = np;
  a.t = int32_t(t);
  a.r = r;
  a.bt = int32_t(bt);
  a.lambda = e->lambda.d();
  a.h2 = e->h2.d();
  a.sigma2 = e->sigma2.d();
  a.s = dx + 8;
  a.w = dx + 8 + r;
  a.lam0 = rg[0];
  e->ex_lam0 = rg[0];
  a.epanel = e->epanel.d();
  a.fpanel = e->fpanel.d();
  gwg::prefer_max_smem(gwg::expsum_e_kernel);
  gwg::expsum_e_kernel<<<r, 256, 0, e->comp>>>(a);
  GWG_CUDA_TRY(cudaGetLastError());
  gwg::prefer_max_smem(gwg::expsum_f_kernel);
  gwg::expsum_f_kernel<<<int(t), 128, 0, e->comp>>>(a);
  GWG_CUDA_TRY(cudaGetLastError());
  e->counters.kernel_launches += 2;
  e->sbr_terms = r;
  return GWG_OK;
}

// E and F for the current traits, once per trait set (both grid paths use them).
int prepare_expsum(gwg_engine* e, gwg_status* st) {
  if (e->expsum_valid) return GWG_OK;
  if (int rc = build_expsum(e, st)) return rc;
  e->expsum_valid = true;
  return GWG_OK;
}

// Trait operands of the split grid: V = [D_j.X_L'_c, D_j.Y'_j] in the padded
// linear-solve layout, W = Z V by the DMMA rotation kernel against Z^T, 8 int8
// slices of W per column, and the D panels of gls_sbr_kernel.
int build_split(gwg_engine* e, gwg_status* st) {
  if (e->split_valid) return GWG_OK;
  NvtxRange nvtx_("build_split");
  using gwg::I8Cfg;
  const int64_t n = e->n, np = e->np, t = e->t, p = e->p;
  const int64_t kp = round_up(n, I8Cfg::BK);
  const int64_t ncols = ceil_div(t, e->lops.kt) * e->lops.rb;  // padded W rows
  if (!e->basis_t_valid) {
    GWG_CUDA_TRY(e->basis_t.ensure(size_t(np) * n * sizeof(double)));
    const dim3 grid(unsigned(ceil_div(n, 32)), unsigned(ceil_div(n, 32)));
    gwg::transpose_kernel<<<grid, dim3(32, 8), 0, e->comp>>>(e->basis.d(), e->basis_t.d(), n, np);
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    e->basis_t_valid = true;
  }
  if (int rc = prepare_expsum(e, st)) return rc;
  // factorised D: only the trait columns of V are rotated, no D panels (for
  // t >= 256: with few traits the small GEMMs cost more than the rotation,
  // c0 0.60 vs 0.71 ms; the choice depends on t only, results stay
  // slab-invariant)
  const bool fact = e->sbr_terms > 0 && p > 1 && t >= 256;
  const bool padded = e->lops.p8 != p || t % e->lops.kt;  // W has padding rows
  const int64_t bt = e->sops.bt;
  const int64_t tiles_t = ceil_div(t, bt);
  GWG_CUDA_TRY(e->dpanel.ensure(size_t(tiles_t) * np * bt * sizeof(double)));
  if (t % bt && !fact)  // padded traits of the last tile contribute zeros
    GWG_CUDA_TRY(cudaMemsetAsync(e->dpanel.d() + size_t(tiles_t - 1) * np * bt, 0,
                                 size_t(np) * bt * sizeof(double), e->comp));
  GWG_CUDA_TRY(e->vmat.ensure(size_t(np) * ncols * sizeof(double)));
  GWG_CUDA_TRY(e->wmat.ensure(size_t(np) * ncols * sizeof(double)));
  if (padded && !fact)
    GWG_CUDA_TRY(cudaMemsetAsync(e->vmat.ptr, 0, size_t(np) * ncols * sizeof(double), e->comp));
  gwg::SplitPrepArgs a;
  a.n = n;
  a.np = np;
  a.t = int32_t(t);
  a.p = int32_t(p);
  a.bt = int32_t(bt);
  a.kt = e->lops.kt;
  a.p8 = e->lops.p8;
  a.rb = e->lops.rb;
  a.lambda = e->lambda.d();
  a.y = e->y_rot.d();
  a.ldy = np;
  a.xl = e->xl_rot.d();
  a.ldxl = np;
  a.h2 = e->h2.d();
  a.sigma2 = e->sigma2.d();
  a.dpanel = e->dpanel.d();
  a.v = e->vmat.d();
  a.y_only = fact ? 1 : 0;
  gwg::prefer_max_smem(gwg::split_prep_kernel);
  gwg::split_prep_kernel<<<int(t), 256, 0, e->comp>>>(a);
  GWG_CUDA_TRY(cudaGetLastError());
  e->counters.kernel_launches += 1;
  if (fact) {
    // W through the factorisation D = E F: the covariate columns
    // W_{j,c} = Z (D_j . X_L'_c) = (Z diag(X_L'_c) E) F_j — one GEMM of inner
    // size n for all c (U = Z [diag(X_L'_c) E]_c, n x r (p-1)), then one of
    // inner size r per c straight into W's padded rows j * p8 + c — instead of
    // rotating t (p-1) columns (n^2 per column); non-negative E and F give the
    // same error bound as Z (D_j . X_L'_c).  The trait column W_{j,p-1} =
    // Z (D_j . Y'_j) is rotated as before.
    const int64_t r = e->sbr_terms, rc_cols = r * (p - 1), p8 = e->lops.p8;
    if (padded)  // padding rows (c >= p, traits past t) stay zero
      GWG_CUDA_TRY(cudaMemsetAsync(e->wmat.ptr, 0, size_t(np) * ncols * sizeof(double), e->comp));
    GWG_CUDA_TRY(e->xepanel.ensure(size_t(np) * rc_cols * sizeof(double)));
    GWG_CUDA_TRY(e->umat.ensure(size_t(n) * rc_cols * sizeof(double)));
    // U's split-K partials: n x r(p-1) outputs over K = n are a few dozen
    // tiles, so K is split until the tiles fill the SMs (summed in a fixed order)
    int ksplit = 1;
    {
      const int64_t kchunks = np / e->sops.bk;
      const int64_t units = ceil_div(n, e->sops.bm) * ceil_div(rc_cols, e->sops.bt);
      while (ksplit < 16 && kchunks % (2 * ksplit) == 0 && kchunks / (2 * ksplit) >= 4 &&
             ceil_div(units * 2 * ksplit, 2) <= e->sms)
        ksplit *= 2;
    }
    if (ksplit > 1)
      GWG_CUDA_TRY(e->upart.ensure(size_t(ksplit) * n * rc_cols * sizeof(double)));
    // The covariate columns (below) and the trait column (a rotation) write
    // disjoint rows of W and share no input but E / F: the covariate chain of
    // small launches runs on the helper stream while this stream rotates.
    if (GWG_COV_STREAM) {
      GWG_CUDA_TRY(cudaEventRecord(e->ev_cov_fork, e->comp));
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->side2, e->ev_cov_fork, 0));
      std::swap(e->comp, e->side2);
    }
    gwg::ExpSumArgs x;
    x.n = n;
    x.np = np;
    x.t = int32_t(t);
    x.r = int32_t(r);
    x.bt = int32_t(e->sops.bt);
    x.lambda = e->lambda.d();
    x.s = e->exps.d() + 8;
    x.w = e->exps.d() + 8 + r;
    x.lam0 = e->ex_lam0;
    x.xmul = e->xl_rot.d();
    x.ldx = np;
    x.ncx = int32_t(p - 1);
    x.panel_out = e->xepanel.d();
    gwg::prefer_max_smem(gwg::expsum_e_kernel);
    gwg::expsum_e_kernel<<<int(rc_cols), 256, 0, e->comp>>>(x);
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    // U[k][(c, q)] = sum_l Z[k][l] x_c[l] E[l][q]  (A = Z^T's columns = Z's rows)
    int rc = sbr_gemm(e, e->basis_t.d(), n, np, n, e->xepanel.d(), np, rc_cols, e->umat.d(),
                      rc_cols, true, st, ksplit, ksplit > 1 ? e->upart.d() : nullptr,
                      n * rc_cols);
    // W[(j p8 + c) np + k] = sum_q U[k][(c, q)] F[q][j]
    for (int64_t c = 0; rc == GWG_OK && c + 1 < p; ++c)
      rc = sbr_gemm(e, e->umat.d() + c * r, r, rc_cols, n, e->fpanel.d(), r, t,
                    e->wmat.d() + c * np, p8 * np, false, st);
    if (GWG_COV_STREAM) {
      std::swap(e->comp, e->side2);
      GWG_CUDA_TRY(cudaEventRecord(e->ev_cov_join, e->side2));
    }
    if (rc == GWG_OK)
      rc = rotate(e, e->vmat.d() + (p - 1) * np, t, e->wmat.d() + (p - 1) * np, st, p8 * np,
                  nullptr, e->basis_t.d(), p8 * np);
    if (GWG_COV_STREAM) GWG_CUDA_TRY(cudaStreamWaitEvent(e->comp, e->ev_cov_join, 0));
    if (rc) return rc;
  } else {
    if (int rc = rotate(e, e->vmat.d(), ncols, e->wmat.d(), st, np, nullptr, e->basis_t.d()))
      return rc;
  }
  if (LIN_FOLD && p > 1) {  // W_j L_j^-T and W_y - W' z_T (split_prep.cuh)
    const gwg::CtxOffsets co = gwg::ctx_offsets(int(p));
    gwg::FoldArgs f;
    f.w = e->wmat.d();
    f.n = n;
    f.np = np;
    f.t = int32_t(t);
    f.p = int32_t(p);
    f.kt = e->lops.kt;
    f.p8 = e->lops.p8;
    f.rb = e->lops.rb;
    f.ctx = e->ctx.d();
    f.stride = co.stride;
    f.z = co.z;
    f.flag = co.flag;
    f.linv = co.linv;
    gwg::prefer_max_smem(gwg::fold_w_kernel);
    gwg::fold_w_kernel<<<int(t), 256, 0, e->comp>>>(f);
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
  }
  GWG_CUDA_TRY(e->wslices.ensure(size_t(I8Cfg::SLICES) * ncols * kp));
  GWG_CUDA_TRY(e->wscale.ensure(size_t(ncols) * sizeof(double)));
  gwg::prefer_max_smem(gwg::slice_basis_kernel);
  gwg::slice_basis_kernel<<<int(ncols), 256, 0, e->comp>>>(e->wmat.d(), np, int32_t(n),
                                                          int32_t(ncols), int32_t(kp),
                                                          static_cast<int8_t*>(e->wslices.ptr),
                                                          e->wscale.d());
  GWG_CUDA_TRY(cudaGetLastError());
  e->counters.kernel_launches += 1;
  e->split_valid = true;
  return GWG_OK;
}

// Split grid over one genotype slab: S_BR on DMMA (gls_sbr_kernel), then the
// exact int8 linear terms + bordered Cholesky (linear_solve_kernel<P>).
// S_BR = (X'.X')^T D for one slab into e->sbr ([trait][SNP], ld ld_s):
// directly against the D panels, or as ((X'.X')^T E) F — two DMMA GEMMs of
// inner size n and r (expsum.cpp).  Needs the E/F panels (build_expsum) or,
// when sbr_terms = 0, the D panels (build_split).  Gated like the launches
// around it (gate_want).
// One gls_sbr_kernel GEMM: dst = A^T P with A (kext x rows, ld lda, read by
// TMA) and P a D-panel operand of K extent pk (a multiple of bk) over `cols`
// columns; dst[j * ldd + i], or dst[i * ldd + j] (rowmajor).  Gated like
// the launches around it (gate_want).
int sbr_gemm(gwg_engine* e, const double* a_op, int64_t kext, int64_t lda, int64_t rows,
             const double* panel, int64_t pk, int64_t cols, double* dst, int64_t ldd,
             bool rowmajor, gwg_status* st, int ksplit, double* partials,
             int64_t split_stride, int64_t pad_chunks) {
  const gwg::SbrOps& so = e->sops;
  CUtensorMap map;
  if (int rc = encode_kmajor(&map, a_op, kext, rows, lda, so.bm, st)) return rc;
  gwg::SbrArgs q;
  q.dpanel = panel;
  q.sbr = dst;
  q.ld = ldd;
  q.rows = rows;
  q.t = int32_t(cols);
  q.tiles_m = int32_t(ceil_div(rows, so.bm));
  q.tiles_t = int32_t(ceil_div(cols, so.bt));
  q.kchunks = int32_t(pk / so.bk + pad_chunks);  // padded chunks: A out of bounds = zeros
  q.np = pk;
  q.rowmajor = rowmajor ? 1 : 0;
  q.gate = gate_word(e);
  q.gate_codes = e->gate_want;
  if (ksplit > 1) {  // partial products into `partials`, summed into dst below
    q.ksplit = ksplit;
    q.sbr = partials;
    q.split_stride = split_stride;
  }
  const int64_t supers = ceil_div(int64_t(q.tiles_m) * q.tiles_t * q.ksplit, 2);
  GWG_CUDA_TRY(so.launch(map, q, int(std::min<int64_t>(supers, e->sms)), e->comp));
  e->counters.kernel_launches += 1;
  if (ksplit > 1) {  // dense dst (ldd = cols, rowmajor) = the partials in order
    gwg::prefer_max_smem(gwg::sum_partials_kernel);
    gwg::sum_partials_kernel<<<int(std::min<int64_t>(ceil_div(split_stride, 256), 4 * e->sms)),
                               256, 0, e->comp>>>(partials, split_stride, ksplit, split_stride,
                                                  dst);
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
  }
  return GWG_OK;
}

int launch_sbr_stage(gwg_engine* e, const double* rot_sq, int64_t rows, int64_t ld_s,
                     gwg_status* st) {
  const int64_t t = e->t;
  GWG_CUDA_TRY(e->sbr.ensure(size_t(ld_s) * t * sizeof(double)));
  auto gemm = [&](const double* a_op, int64_t kext, int64_t lda, const double* panel,
                  int64_t pk, int64_t cols, double* dst, int64_t ldd, bool rowmajor) {
    return sbr_gemm(e, a_op, kext, lda, rows, panel, pk, cols, dst, ldd, rowmajor, st);
  };
  e->counters.sbr_terms = e->sbr_terms;
  e->counters.sbr_flops += uint64_t(rows) * 2ull *
                           (e->sbr_terms ? uint64_t(e->sbr_terms) * uint64_t(e->n + t)
                                         : uint64_t(e->n) * uint64_t(t));
  if (const int64_t r = e->sbr_terms) {
    GWG_CUDA_TRY(e->gmat.ensure(size_t(rows) * r * sizeof(double)));
    // G = (X'.X')^T E has only r = 64..512 columns: a slab of a few thousand
    // SNPs is a few dozen tiles (config 2's default 3,000-SNP slab: 24 CTAs,
    // 0.65 ms per slab, a quarter of the streamed run's grid time).  From
    // K >= 2048 on, K is split into up to 8 parts of >= 32 chunks, summed in a
    // fixed order.  The split depends on n alone, never on the slab, so results
    // stay bitwise independent of the slab width; below 2048 nothing changes.
    int ksplit = 1;
    const int64_t kchunks = e->np / e->sops.bk;
    while (ksplit < 8 && ceil_div(kchunks, int64_t(2 * ksplit)) >= 32) ksplit *= 2;
    if (ksplit > 1) {
      const int64_t kc_per = ceil_div(kchunks, int64_t(ksplit));
      GWG_CUDA_TRY(e->gpart.ensure(size_t(ksplit) * rows * r * sizeof(double)));
      if (int rc = sbr_gemm(e, rot_sq, e->n, e->np, rows, e->epanel.d(), e->np, r, e->gmat.d(), r,
                            true, st, ksplit, e->gpart.d(), rows * r, kc_per * ksplit - kchunks))
        return rc;
    } else if (int rc = gemm(rot_sq, e->n, e->np, e->epanel.d(), e->np, r, e->gmat.d(), r, true)) {
      return rc;
    }
    return gemm(e->gmat.d(), r, r, e->fpanel.d(), r, t, e->sbr.d(), ld_s, false);
  }
  return gemm(rot_sq, e->n, e->np, e->dpanel.d(), e->np, t, e->sbr.d(), ld_s, false);
}

// The trait-side operands of the split grid (W, its slices, E/F) depend only
// on the spectrum and the traits.  When they are due, mark the fork point on
// the compute stream before the SNP-side work of the slab (its upload and
// rotation) is queued: launch_split then builds them on the side stream from
// that point on — concurrently with the SNP side — and the compute stream
// joins before the S_BR stage.  Only below 16 K stages (n <= 1920), where the
// trait-side build is small next to the HBM-bound SNP conversion it overlaps:
// measured step c0 0.554 -> 0.540 ms, c1 4.43 -> 4.39, p = 12 6.50 -> 6.45;
// at n = 10,000 the W build (8e11 flop) slowed the concurrent rotation 43.9 ->
// 55.1 ms (step 87.9 -> 89.8), at n = 2000 (c4) 39.6 -> 40.4.
int mark_trait_fork(gwg_engine* e, bool rotated_input, gwg_status* st) {
  e->fork_pending = false;
  if (!e->split || e->split_valid || rotated_input || e->snp_coding == GWG_SNP_REAL ||
      e->n >= kMaxGenotypeN || e->t <= 0 || pair_mma_default(round_up(e->n, gwg::I8Cfg::BK)))
    return GWG_OK;
  // traits still queued on the side stream: the build follows them there
  if (!e->side_pending) GWG_CUDA_TRY(cudaEventRecord(e->ev_fork, e->comp));
  e->fork_pending = true;
  return GWG_OK;
}

// Before the persistent SNP rotation takes every SM: queue the split grid's
// trait-side build (W, its slices, E/F) on the side stream — behind the
// trait work gwg_set_traits left there, or from the fork point — and join.
// The trait side then overlaps the slab's upload and HBM-bound code
// conversion instead of queueing behind the rotation (its small kernels find
// no free SM while the rotation runs).  The build is ungated: the operands
// belong to the traits, not to this slab, so a first slab that takes the FP64
// path under GWG_SNP_AUTO cannot leave a stale W marked valid.
int split_build_ahead(gwg_engine* e, gwg_status* st) {
  if (e->fork_pending && !e->split_valid) {
    e->fork_pending = false;
    if (!e->side_pending) GWG_CUDA_TRY(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
    const int saved_gate = e->gate_want;
    e->gate_want = -1;
    std::swap(e->comp, e->side);
    const int rc = build_split(e, st);
    std::swap(e->comp, e->side);
    e->gate_want = saved_gate;
    e->side_pending = true;  // joined below even when the build failed part-way
    if (rc) {
      join_side(e);
      return rc;
    }
  }
  if (e->side_pending && e->join_ev) {
    GWG_CUDA_TRY(cudaEventRecord(e->join_ev[0], e->comp));
    GWG_CUDA_TRY(join_side(e));
    GWG_CUDA_TRY(cudaEventRecord(e->join_ev[1], e->comp));
    *e->join_timed = true;
    return GWG_OK;
  }
  GWG_CUDA_TRY(join_side(e));
  return GWG_OK;
}

int launch_split(gwg_engine* e, const double* rot_sq, int64_t rows, int64_t i0, int64_t m_total,
                 double* dev_out, int64_t out_si, int64_t out_sj, gwg_status* st) {
  {
    // The trait-derived operands (W, its slices, E/F) belong to the traits,
    // not to this slab: they are built ungated, so a first slab that takes the
    // FP64 path under GWG_SNP_AUTO cannot leave a stale W marked valid.
    int rc;
    if (e->fork_pending && !e->split_valid) {  // on the side stream from the fork point
      rc = split_build_ahead(e, st);
    } else {
      GWG_CUDA_TRY(join_side(e));
      const int saved_gate = e->gate_want;
      e->gate_want = -1;
      rc = build_split(e, st);
      e->gate_want = saved_gate;
    }
    if (rc) return rc;
  }
  using gwg::I8Cfg;
  const int64_t t = e->t, p = e->p;
  const int64_t kp = round_up(e->n, I8Cfg::BK);
  const int64_t tiles_r = ceil_div(t, e->lops.kt);
  const int64_t ncols = tiles_r * e->lops.rb;
  const int64_t ld_s = round_up(rows, 2);

  // ---- S_BR ----
  cudaEvent_t* sev = e->split_ev ? e->split_ev : e->ev_s;
  GWG_CUDA_TRY(cudaEventRecord(sev[0], e->comp));
  if (int rc = launch_sbr_stage(e, rot_sq, rows, ld_s, st)) return rc;
  GWG_CUDA_TRY(cudaEventRecord(sev[1], e->comp));

  // ---- linear terms (int8 tcgen05) + solve ----
  // CTA pairs multicasting the W-slice tile (measured: c1 2.90 -> 2.86 ms,
  // c2 22.5 -> 20.9, c4 43.1 -> 40.4).  GWG_OPT_I8_CLUSTER = 1|2|3 forces single
  // CTAs / these B pairs / pairs on two W tiles multicasting the SNP tile —
  // the last measured slower even with one or two traits per tile (c4 33.2
  // -> 35.6 ms, p = 12 5.25 -> 5.62), so the SNP tile's L2 traffic is not
  // what bounds those configs.
  // GWG_OPT_I8_CLUSTER = 4: pairs running one cta_group::2 MMA (32-row W
  // tiles; other tilings take the B pairs)
  int cl = e->i8_cluster ? e->i8_cluster : pair_mma_default(kp) ? 4 : 2;
  if (cl == 4 && !e->lops.launch[3]) cl = 2;
  CUtensorMap tx, tw, tout, twh;
  if (int rc = encode_i8(&tx, e->xi8.ptr, kp, rows, &tw, e->wslices.ptr, ncols, e->lops.rb,
                         e->lops.b_slices_box[cl - 1], st, e->lops.a_box_rows[cl - 1], &twh))
    return rc;
  // numpy layout with a 16-byte pitch and base: results leave by TMA store;
  // stream layout ((j*ldo + i)*p, out_si = 1) by TMA boxes {32p, cells} when
  // the trait pitch is 16-byte aligned
  const bool aligned = (reinterpret_cast<uintptr_t>(dev_out) & 15) == 0;
  const bool aligned32 = (reinterpret_cast<uintptr_t>(dev_out) & 31) == 0;
  // no staging tiles (p % 4 == 0): 256-bit stores in either layout, scalar
  // stores for a base that is not 32-byte aligned; tout is the S_BR map
  const bool nostage = e->lops.nostage;
  const int use_tma = nostage ? (aligned32 ? 3 : 0)
                      : (out_sj == 1 && (out_si * p) % 2 == 0 && aligned) ? 1
                      : (out_si == 1 && LIN_STREAM_STG && e->lops.stream_stg && aligned32 &&
                         (out_sj * p) % 4 == 0) ? 3
                      : (out_si == 1 && e->lops.stream_tma && (out_sj * p) % 2 == 0 && aligned &&
                         LIN_STREAM_TMA) ? 2 : 0;
  {
    auto encode = get_encode();
    CUresult r;
    if (e->lops.sbr_tma) {
      // S_BR [trait][SNP] (ld ld_s, even): one {BM SNPs, KT traits} box per tile
      const cuuint64_t gdim[2] = {cuuint64_t(rows), cuuint64_t(t)};
      const cuuint64_t gstride[1] = {cuuint64_t(ld_s * 8)};
      const cuuint32_t box[2] = {cuuint32_t(I8Cfg::BM), cuuint32_t(e->lops.kt)};
      const cuuint32_t es[2] = {1, 1};
      r = encode(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, e->sbr.d(), gdim, gstride, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return set_status(st, GWG_CUDA, -1, -1, "tensor map (S_BR) failed (%d)", int(r));
    } else if (use_tma == 2) {
      const cuuint64_t gdim[2] = {cuuint64_t(rows * p), cuuint64_t(t)};
      const cuuint64_t gstride[1] = {cuuint64_t(out_sj * p * 8)};
      const cuuint32_t box[2] = {cuuint32_t(32 * p), cuuint32_t(e->lops.stream_rows)};
      const cuuint32_t es[2] = {1, 1};
      r = encode(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dev_out, gdim, gstride, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t gdim[2] = {cuuint64_t(t * p), cuuint64_t(rows)};
      const cuuint64_t gstride[1] = {cuuint64_t(use_tma ? out_si * p * 8 : 16)};
      // 16-double swizzled chunks, or one unswizzled {row, 32} box per warp tile
      const bool tma_row = e->lops.tma_row;
      const cuuint32_t box[2] = {tma_row ? cuuint32_t(e->lops.row) : gwg::I8Cfg::OUT_Q, 32};
      const cuuint32_t es[2] = {1, 1};
      r = encode(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dev_out, gdim, gstride, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                 tma_row ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if ((use_tma == 1 || use_tma == 2) && r != CUDA_SUCCESS)
      return set_status(st, GWG_CUDA, -1, -1, "tensor map (results) failed (%d)", int(r));
  }
  gwg::LinArgs a;
  a.scale = e->wscale.d();
  a.sbr = e->sbr.d();
  a.ld_s = ld_s;
  a.ctx = e->ctx.d();
  a.out = dev_out;
  a.out_si = out_si;
  a.out_sj = out_sj;
  a.use_tma = use_tma;
  a.t = int32_t(t);
  a.rows = rows;
  a.i0 = i0;
  a.m_total = m_total;
  a.tiles_m = int32_t(ceil_div(rows, I8Cfg::BM));
  a.tiles_r = int32_t(tiles_r);
  a.kstages = int32_t(kp / I8Cfg::BK);
  a.b_resident = size_t(I8Cfg::SLICES) * ncols * kp <= (size_t(GWG_B_RESIDENT_MB) << 20);
  a.gate = gate_word(e);
  a.gate_codes = e->gate_want;
  // numpy-order results with L2-resident W slices: trait tiles fastest, so
  // the tiles in flight write contiguous rows of b (I8Sched raster)
  a.raster = (LIN_RASTER == 2 || (LIN_RASTER == 1 && out_sj == 1 && a.b_resident)) ? 1 : 0;
  a.err_key = static_cast<unsigned long long*>(e->err.ptr) + 1;
  const int64_t tiles = int64_t(a.tiles_m) * a.tiles_r;
  (void)tiles;
  GWG_CUDA_TRY(e->lops.launch[cl - 1](tx, tw, tout, a, e->sms, e->comp, twh));
  GWG_CUDA_TRY(cudaEventRecord(sev[2], e->comp));
  e->split_timed = true;
  e->counters.kernel_launches += 1;
  return GWG_OK;
}

// Grid kernel over one rotated slab (rot, rot_sq: ld np, `rows` SNPs) into dev_out.
int launch_slab(gwg_engine* e, const double* rot, const double* rot_sq, int64_t rows, int64_t i0,
                int64_t m_total, double* dev_out, int64_t out_si, int64_t out_sj,
                gwg_status* st) {
  GWG_CUDA_TRY(join_side(e));  // the grid reads the trait operands
  const uint64_t cells = uint64_t(rows) * uint64_t(e->t);
  e->counters.grid_flops += cells * 2ull * uint64_t(e->n) * uint64_t(e->p + 1);
  e->counters.loop_flops += cells * uint64_t(e->n) * (5 + 2 * uint64_t(e->p - 1));
  if (e->slab_auto) {  // both paths queued, each gated on the slab's verdict
    e->gate_want = e->split ? 1 : -1;
    int rc = e->split ? launch_split(e, rot_sq, rows, i0, m_total, dev_out, out_si, out_sj, st)
                      : GWG_OK;
    e->gate_want = e->split ? 0 : -1;
    if (rc == GWG_OK) rc = launch_fused(e, rot, rot_sq, rows, i0, m_total, dev_out, out_si, out_sj, st);
    e->gate_want = -1;
    return rc;
  }
  if (e->slab_i8 && e->split)
    return launch_split(e, rot_sq, rows, i0, m_total, dev_out, out_si, out_sj, st);
  return launch_fused(e, rot, rot_sq, rows, i0, m_total, dev_out, out_si, out_sj, st);
}

// The all-FP64 fused grid kernel over one rotated slab.
int launch_fused(gwg_engine* e, const double* rot, const double* rot_sq, int64_t rows, int64_t i0,
                 int64_t m_total, double* dev_out, int64_t out_si, int64_t out_sj,
                 gwg_status* st) {
  if (!e->bops_valid) {  // the panels gwg_set_traits skipped (contexts are rebuilt alike)
    gwg::PrepArgs pa = e->prep_args;
    pa.panels = 1;
    GWG_CUDA_TRY(e->ops.prep(pa, e->comp));
    e->counters.kernel_launches += 1;
    e->bops_valid = true;
  }
  CUtensorMap map, map_sq;
  if (int rc = encode_kmajor(&map, rot, e->n, rows, e->np, e->ops.bm, st)) return rc;
  if (int rc = encode_kmajor(&map_sq, rot_sq, e->n, rows, e->np, e->ops.bm, st)) return rc;
  gwg::GridArgs a;
  a.bops = e->bops.d();
  a.ctx = e->ctx.d();
  a.out = dev_out;
  a.out_si = out_si;
  a.out_sj = out_sj;
  a.rows = rows;
  a.i0 = i0;
  a.m_total = m_total;
  a.t = int32_t(e->t);
  a.tiles_m = int32_t(ceil_div(rows, e->ops.bm));
  a.tiles_t = int32_t(ceil_div(e->t, e->ops.bt));
  a.kchunks = int32_t(e->np / e->ops.bk);
  a.np = e->np;
  a.err_key = static_cast<unsigned long long*>(e->err.ptr) + 1;
  a.gate = gate_word(e);
  a.gate_codes = e->gate_want;
  const int64_t tiles = int64_t(a.tiles_m) * a.tiles_t;
  const int ctas = int(std::min<int64_t>(tiles, e->sms));
  // S_BR through the factorised D (two DMMA GEMMs on X'.X'), then the grid
  // kernel without the D column and the X'.X' operand (GridCfg::EXT): 2np
  // instead of 2n(p+1) flop per cell (GWG_OPT_REAL_SPLIT = 0 keeps the single
  // fused kernel).  Measured per step (fused -> split): c1 36.0 -> 32.3 ms,
  // c3 150 -> 127, c4 297 -> 287, p = 8 32.9 -> 30.7, p = 12 48.4 -> 46.3;
  // few traits keep the fused kernel (c0, t = 100: 1.26 vs 1.39 ms) — the
  // choice depends on t only, so results stay bitwise independent of slabs.
  if (e->real_split && e->lowrank && e->t >= 256) {
    {
      const int saved_gate = e->gate_want;  // trait operands: ungated (see launch_split)
      e->gate_want = -1;
      const int rc = prepare_expsum(e, st);
      e->gate_want = saved_gate;
      if (rc) return rc;
    }
    if (e->sbr_terms > 0) {
      const int64_t ld_s = round_up(rows, 2);
      if (int rc = launch_sbr_stage(e, rot_sq, rows, ld_s, st)) return rc;
      a.sbr = e->sbr.d();
      a.ld_s = ld_s;
      GWG_CUDA_TRY(e->ops.grid_ext(map, map_sq, a, ctas, e->comp));
      e->counters.kernel_launches += 1;
      return GWG_OK;
    }
  }
  GWG_CUDA_TRY(e->ops.grid(map, map_sq, a, ctas, e->comp));
  e->counters.kernel_launches += 1;
  return GWG_OK;
}

int square_rotated(gwg_engine* e, int64_t cols, gwg_status* st) {
  e->slab_i8 = false;
  e->slab_auto = false;
  GWG_CUDA_TRY(gwg::launch_square(e->rot.d(), e->rot_sq.d(), size_t(e->np) * cols, e->comp));
  e->counters.kernel_launches += 1;
  return GWG_OK;
}

// Default streamed slab: ~96 MB of results per slab, in whole waves of the
// persistent FP64 grid kernel (tiles_m * tiles_t a multiple of the SM count)
// when a wave is that small; with many traits (a wave's results would be
// tens of GB, c3: 3.2 MB per SNP) a multiple of 128 SNPs — the int8 kernels'
// SNP tile — with at least 128.
int64_t default_slab(const gwg_engine* e, int64_t m) {
  const int64_t tiles_t = ceil_div(e->t, int64_t(e->ops.bt) * e->ops.groups);
  const int64_t unit_tiles = e->sms / std::gcd<int64_t>(tiles_t, e->sms);
  const int64_t unit = unit_tiles * e->ops.bm;  // SNPs per whole-wave slab
  const int64_t target = std::max<int64_t>(1, (96ll << 20) / (e->t * e->p * 8));
  if (target >= unit) return std::min(m, target / unit * unit);
  return std::min(m, std::max<int64_t>(128, target / 128 * 128));
}

// memcpy split over a few threads for large slabs (pageable user memory <->
// pinned staging).
void parallel_copy(void* dst, const void* src, size_t bytes) {
  const size_t kChunk = size_t(8) << 20;
  const int threads = int(std::min<size_t>(8, (bytes + kChunk - 1) / kChunk));
  if (threads <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> pool;
  const size_t part = (bytes + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    const size_t lo = size_t(w) * part, hi = std::min(bytes, lo + part);
    if (lo >= hi) break;
    pool.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    });
  }
  for (auto& th : pool) th.join();
}

int raise_cell_error(gwg_engine* e, gwg_status* st) {
  const unsigned long long key = e->err_host[1];
  if (key == ~0ull) return GWG_OK;
  const int64_t j = int64_t(key / uint64_t(kKeyStride));
  const int64_t i = int64_t(key % uint64_t(kKeyStride));
  return set_status(st, GWG_NOT_POSITIVE_DEFINITE, i, j,
                    "normal equations are not positive definite at cell (variant %lld, trait "
                    "%lld)",
                    (long long)i, (long long)j);
}


// ---- shared-operand installs ------------------------------------------------

int set_spectrum_impl(gwg_engine* e, const double* basis, int64_t ldb, const double* lambda,
                      int where, gwg_status* st) {
  if (!basis || !lambda) return set_status(st, GWG_DIMENSION, -1, -1, "null spectrum operand");
  if (int rc = upload_cols(e, e->basis, basis, ldb, e->n, where, e->comp, st)) return rc;
  if (int rc = upload(e, e->lambda, lambda, size_t(e->n), where, st)) return rc;
  if (int rc = spectrum_range(e, st)) return rc;
  e->have_spectrum = true;
  e->have_covariates = false;
  e->have_traits = false;
  invalidate_derived(e, true);
  return GWG_OK;
}

int set_covariates_impl(gwg_engine* e, const double* xl, int64_t ldx, int where, bool rotated,
                        gwg_status* st) {
  if (!e->have_spectrum)
    return set_status(st, GWG_DIMENSION, -1, -1, "gwg_set_spectrum must come first");
  const int64_t pm1 = e->p - 1;
  GWG_CUDA_TRY(e->xl_rot.ensure(size_t(e->np) * std::max<int64_t>(pm1, 1) * sizeof(double)));
  if (pm1 > 0) {
    if (!xl) return set_status(st, GWG_DIMENSION, -1, -1, "null covariate block");
    if (rotated) {
      if (int rc = upload_cols(e, e->xl_rot, xl, ldx, pm1, where, e->comp, st)) return rc;
    } else {
      if (int rc = upload_cols(e, e->xl_raw, xl, ldx, pm1, where, e->comp, st)) return rc;
      if (int rc = rotate(e, e->xl_raw.d(), pm1, e->xl_rot.d(), st)) return rc;
    }
  }
  if (where != GWG_DEVICE)  // the caller may free or reuse its host block on return
    GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));
  e->have_covariates = true;
  e->have_traits = false;
  invalidate_derived(e, false);
  return GWG_OK;
}

// Traits: Y (raw or rotated, leading dimension ldy, on y_where) and h2/sigma2
// (on s_where).  Nothing here waits for the device: the weight-floor verdict
// stays in error word 0 until the next synchronising call reads it.
int set_traits_body(gwg_engine* e, int64_t t, const double* y, int64_t ldy, int y_where,
                    const double* h2, const double* sigma2, int s_where, bool rotated,
                    gwg_status* st) {
  if (!e->have_covariates)
    return set_status(st, GWG_DIMENSION, -1, -1, "gwg_set_covariates must come first");
  if (t < 1 || t > (int64_t(1) << 30))
    return set_status(st, GWG_DIMENSION, -1, -1, "trait count out of range (got %lld)",
                      (long long)t);
  if (!y || !h2 || !sigma2) return set_status(st, GWG_DIMENSION, -1, -1, "null trait operand");
  e->have_traits = false;
  invalidate_derived(e, false);
  const int64_t n = e->n;
  if (int rc = upload(e, e->h2, h2, size_t(t), s_where, st)) return rc;
  if (int rc = upload(e, e->sigma2, sigma2, size_t(t), s_where, st)) return rc;
  e->traits_host_valid = s_where == GWG_HOST;
  e->range_pending = false;
  if (e->traits_host_valid) {
    e->h2_host.assign(h2, h2 + t);
    e->s2_host.assign(sigma2, sigma2 + t);
  } else if (e->lowrank && (e->snp_coding == GWG_SNP_REAL ? e->real_split : true)) {
    // queue the exponential sum's range first (it needs only lambda, h2 and
    // sigma2): the Y rotation and the context build queued behind it keep the
    // device busy while the 48-byte answer travels, so the split grid's
    // build finds it on the host without stalling the device
    GWG_CUDA_TRY(e->exps.ensure(size_t(8 + 2 * 512) * sizeof(double)));
    gwg::prefer_max_smem(gwg::expsum_range_kernel);
    gwg::expsum_range_kernel<<<1, 256, 0, e->comp>>>(e->lambda.d(), e->n, e->h2.d(),
                                                      e->sigma2.d(), int32_t(t), e->exps.d());
    GWG_CUDA_TRY(cudaGetLastError());
    e->counters.kernel_launches += 1;
    GWG_CUDA_TRY(cudaMemcpyAsync(e->range_host, e->exps.d(), 6 * sizeof(double),
                                 cudaMemcpyDeviceToHost, e->comp));
    GWG_CUDA_TRY(cudaEventRecord(e->ev_range, e->comp));
    e->range_pending = true;
  }
  bool uploads_done = false;  // ev_traits_in follows every host upload of this call
  if (rotated) {
    if (int rc = upload_cols(e, e->y_rot, y, ldy, t, y_where, e->comp, st)) return rc;
    GWG_CUDA_TRY(cudaEventRecord(e->ev_traits_in, e->comp));
    uploads_done = true;
  } else {
    // Y on this device in a TMA-addressable layout (even pitch, 16-byte
    // aligned) is rotated where it lies — read asynchronously, like every
    // device operand — instead of through a copy
    bool in_place = false;
    if (y_where == GWG_DEVICE && ldy % 2 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
      cudaPointerAttributes pa{};
      in_place = cudaPointerGetAttributes(&pa, y) == cudaSuccess &&
                 pa.type == cudaMemoryTypeDevice && pa.device == e->device;
      (void)cudaGetLastError();
    }
    GWG_CUDA_TRY(e->y_rot.ensure(size_t(e->np) * t * sizeof(double)));
    if (in_place) {
      if (int rc = rotate(e, y, t, e->y_rot.d(), st, ldy)) return rc;
    } else {
      // pitch n when TMA can address it (n even): one flat copy for a
      // contiguous Y instead of a pitched one
      const int64_t ldr = raw_ld(e);
      if (int rc = upload_cols(e, e->y_raw, y, ldy, t, y_where, e->comp, st, ldr)) return rc;
      GWG_CUDA_TRY(cudaEventRecord(e->ev_traits_in, e->comp));
      uploads_done = true;
      if (int rc = rotate(e, e->y_raw.d(), t, e->y_rot.d(), st, ldr)) return rc;
    }
  }
  const int64_t tiles_t = ceil_div(t, e->ops.bt);
  const size_t bops_doubles = size_t(tiles_t) * e->np * (e->p + 1) * e->ops.bt;
  GWG_CUDA_TRY(e->bops.ensure(bops_doubles * sizeof(double)));
  GWG_CUDA_TRY(e->ctx.ensure(size_t(t) * e->ops.ctx_stride * sizeof(double)));
  if (t % e->ops.bt)  // padded traits of the last tile contribute zeros
    GWG_CUDA_TRY(cudaMemsetAsync(e->bops.d() + size_t(tiles_t - 1) * e->np * (e->p + 1) *
                                                   e->ops.bt,
                                 0, size_t(e->np) * (e->p + 1) * e->ops.bt * sizeof(double),
                                 e->comp));
  GWG_CUDA_TRY(cudaMemsetAsync(e->err.ptr, 0xff, sizeof(unsigned long long), e->comp));
  gwg::PrepArgs a;
  a.n = n;
  a.np = e->np;
  a.t = int32_t(t);
  a.lambda = e->lambda.d();
  a.y = e->y_rot.d();
  a.ldy = e->np;
  a.xl = e->xl_rot.d();
  a.ldxl = e->np;
  a.h2 = e->h2.d();
  a.sigma2 = e->sigma2.d();
  a.bops = e->bops.d();
  a.ctx = e->ctx.d();
  a.trait_err = static_cast<unsigned long long*>(e->err.ptr);
  // explicit genotype coding with the split grid never reads the FP64 grid's
  // operand panels unless a pre-rotated slab arrives: built on demand then
  // (launch_fused)
  a.panels = (e->snp_coding == GWG_SNP_GENOTYPES && e->split) ? 0 : 1;
  e->bops_valid = a.panels != 0;
  e->prep_args = a;
  GWG_CUDA_TRY(e->ops.prep(a, e->comp));
  e->counters.kernel_launches += 1;
  e->counters.context_builds += 1;
  const uint64_t pm1 = uint64_t(e->p - 1);
  e->counters.loop_flops += uint64_t(t) * uint64_t(n) * (5 + 3 * pm1 + pm1 * pm1);
  // host operands are consumed before the call returns (the caller owns and
  // may reuse them, like the reference's synchronous load_pass); device
  // operands stay asynchronous
  // (the uploads, not the context build: the caller may reuse its buffers, the
  // device work continues asynchronously)
  if (y_where == GWG_HOST || s_where == GWG_HOST) {
    if (uploads_done)
      GWG_CUDA_TRY(cudaEventSynchronize(e->ev_traits_in));  // after every upload
    else
      GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));
  }
  e->t = t;
  e->have_traits = true;
  return GWG_OK;
}

// gwg_set_traits: on the split path (genotype / auto coding at the sizes
// that fork the split build, mark_trait_fork) the trait work — uploads, the
// Y rotation, the exponential sum's range, the contexts — is queued on the
// side stream from this point of the compute stream, so it overlaps the next
// slab's upload and code conversion; whatever reads it joins first
// (join_side).  Elsewhere it runs on the compute stream.
int set_traits_impl(gwg_engine* e, int64_t t, const double* y, int64_t ldy, int y_where,
                    const double* h2, const double* sigma2, int s_where, bool rotated,
                    gwg_status* st) {
  const bool on_side = GWG_TRAITS_ON_SIDE && e->split && e->snp_coding != GWG_SNP_REAL &&
                       e->n < kMaxGenotypeN && !pair_mma_default(round_up(e->n, gwg::I8Cfg::BK));
  if (!on_side) {
    GWG_CUDA_TRY(join_side(e));
    return set_traits_body(e, t, y, ldy, y_where, h2, sigma2, s_where, rotated, st);
  }
  if (!e->side_pending) {  // the side stream starts from here
    GWG_CUDA_TRY(cudaEventRecord(e->ev_fork, e->comp));
    GWG_CUDA_TRY(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
  }
  e->side_pending = true;
  std::swap(e->comp, e->side);
  const int rc = set_traits_body(e, t, y, ldy, y_where, h2, sigma2, s_where, rotated, st);
  std::swap(e->comp, e->side);
  return rc;
}

}  // namespace gwg_host

using namespace gwg_host;

extern "C" {

const char* gwg_version(void) { return "gwgrid_cuda 0.2.0 sm_100a"; }

uint64_t gwg_cell_hash(int64_t i, int64_t j, int64_t c, uint64_t bits) {
  return gwg::cell_term(gwg::cell_key(uint64_t(i), uint64_t(j)), uint64_t(c), bits);
}

gwg_engine* gwg_engine_create(int32_t device, int64_t n, int64_t p, gwg_status* st) {
  clear_status(st);
  if (n < 1 || p < 1 || p > n) {
    set_status(st, GWG_DIMENSION, -1, -1, "bad dimensions n=%lld p=%lld", (long long)n,
               (long long)p);
    return nullptr;
  }
  if (n > (int64_t(1) << 28)) {
    set_status(st, GWG_DIMENSION, -1, -1, "n too large");
    return nullptr;
  }
  KernelOps ops;
  gwg::LinOps lops;
  if (!gwg::ops_for(p, &ops) || !gwg::lin_ops_for(p, &lops)) {
    set_status(st, GWG_DIMENSION, -1, -1,
               "p=%lld is outside the compiled predictor range 1..32", (long long)p);
    return nullptr;
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
    cudaGetLastError();
    set_status(st, GWG_CUDA, -1, -1, "CUDA device %d not available", device);
    return nullptr;
  }
  auto* e = new gwg_engine();
  e->device = device;
  e->n = n;
  e->p = p;
  e->np = round_up(n, kBK);
  e->ops = ops;
  e->lops = lops;
  // The numerics are fixed by the engine's options alone (gwg_set_option),
  // never by the caller's environment.
  e->sops = gwg::sbr_ops(0);
  auto bail = [&](const char* what, cudaError_t err) {
    set_status(st, GWG_CUDA, -1, -1, "%s: %s", what, cudaGetErrorString(err));
    gwg_engine_destroy(e);
    return nullptr;
  };
  cudaError_t err;
  if ((err = cudaSetDevice(device)) != cudaSuccess) return bail("cudaSetDevice", err);
  cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, device);
  if (GWG_PERSIST_L2_MB > 0) {
    // L2 set-aside for the evict_last operands (the W / Z slices the int8
    // kernels keep resident): without one, evict_last lines compete with the
    // streamed results like any other
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    const size_t want = std::min<size_t>(size_t(max_persist), size_t(GWG_PERSIST_L2_MB) << 20);
    if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    (void)cudaGetLastError();
  }
  int cc_major = 0;
  cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device);
  if (cc_major != 10) {
    set_status(st, GWG_CUDA, -1, -1, "device %d has compute capability %d.x; sm_100a required",
               device, cc_major);
    gwg_engine_destroy(e);
    return nullptr;
  }
  if ((err = cudaStreamCreateWithFlags(&e->comp, cudaStreamNonBlocking)) != cudaSuccess)
    return bail("stream", err);
  if ((err = cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking)) != cudaSuccess)
    return bail("stream", err);
  if ((err = cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking)) != cudaSuccess)
    return bail("stream", err);
  {
    // the side stream (trait-side split build) at the highest priority: its
    // small kernels take SMs as the HBM-bound SNP conversion's blocks drain,
    // instead of queueing behind it and the persistent rotation
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if ((err = cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking,
                                            GWG_SIDE_PRIORITY ? greatest : least)) != cudaSuccess)
      return bail("stream", err);
  }
  {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if ((err = cudaStreamCreateWithPriority(&e->side2, cudaStreamNonBlocking,
                                            GWG_SIDE_PRIORITY ? greatest : least)) != cudaSuccess)
      return bail("stream", err);
  }
  cudaEventCreateWithFlags(&e->ev_cov_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_traits_in, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_cov_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming);
  for (int b = 0; b < 2; ++b) {
    cudaEventCreateWithFlags(&e->ev_h2d[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e->ev_rot_done[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e->ev_comp[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e->ev_d2h_done[b], cudaEventDisableTiming);
  }
  cudaEventCreate(&e->ev_k0);
  cudaEventCreate(&e->ev_k1);
  cudaEventCreate(&e->ev_r0);
  cudaEventCreate(&e->ev_r1);
  for (cudaEvent_t& ev : e->ev_s) cudaEventCreate(&ev);
  if ((err = e->err.ensure(3 * sizeof(unsigned long long))) != cudaSuccess)
    return bail("cudaMalloc", err);
  if ((err = cudaMemsetAsync(e->err.ptr, 0xff, 3 * sizeof(unsigned long long), e->comp)) !=
      cudaSuccess)
    return bail("cudaMemset", err);
  if ((err = cudaMallocHost(&e->err_host, 3 * sizeof(unsigned long long))) != cudaSuccess)
    return bail("cudaMallocHost", err);
  if ((err = cudaMallocHost(&e->range_host, 8 * sizeof(double))) != cudaSuccess)
    return bail("cudaMallocHost", err);
  cudaEventCreateWithFlags(&e->ev_range, cudaEventDisableTiming);
  return e;
}

void gwg_engine_destroy(gwg_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->comp) cudaStreamSynchronize(e->comp);
  if (e->h2d) cudaStreamSynchronize(e->h2d);
  if (e->d2h) cudaStreamSynchronize(e->d2h);
  if (e->side) cudaStreamSynchronize(e->side);
  if (e->side2) cudaStreamSynchronize(e->side2);
  for (DevBuf* b : {&e->basis, &e->lambda, &e->xl_raw, &e->xl_rot, &e->y_raw, &e->y_rot, &e->h2,
                    &e->sigma2, &e->bops, &e->ctx, &e->raw[0], &e->raw[1], &e->rot, &e->rot_sq, &e->out[0],
                    &e->out[1], &e->stage, &e->err, &e->zslices, &e->zscale, &e->xi8, &e->basis_t, &e->vmat, &e->wmat,
                    &e->wslices, &e->wscale, &e->dpanel, &e->sbr, &e->epanel, &e->fpanel,
                    &e->gmat, &e->gpart, &e->exps, &e->xepanel, &e->umat, &e->upart, &e->raw8[0], &e->raw8[1], &e->csum})
    b->release();
  if (e->err_host) cudaFreeHost(e->err_host);
  if (e->range_host) cudaFreeHost(e->range_host);
  if (e->ev_range) cudaEventDestroy(e->ev_range);
  for (int b = 0; b < 2; ++b) {
    if (e->ev_h2d[b]) cudaEventDestroy(e->ev_h2d[b]);
    if (e->ev_rot_done[b]) cudaEventDestroy(e->ev_rot_done[b]);
    if (e->ev_comp[b]) cudaEventDestroy(e->ev_comp[b]);
    if (e->ev_d2h_done[b]) cudaEventDestroy(e->ev_d2h_done[b]);
  }
  for (cudaEvent_t ev : {e->ev_k0, e->ev_k1, e->ev_r0, e->ev_r1, e->ev_s[0], e->ev_s[1], e->ev_s[2],
                         e->ev_wait, e->ev_signal, e->ev_fork, e->ev_join, e->ev_cov_fork,
                         e->ev_cov_join, e->ev_traits_in})
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e->slab_events) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e->pipe_events) cudaEventDestroy(ev);
  for (auto& tm : e->timings)
    for (cudaEvent_t ev : tm.ev)
      if (ev) cudaEventDestroy(ev);
  for (PinBuf& b : e->pin_x) b.release();
  for (PinBuf& b : e->pin_res) b.release();
  if (e->comp) cudaStreamDestroy(e->comp);
  if (e->h2d) cudaStreamDestroy(e->h2d);
  if (e->d2h) cudaStreamDestroy(e->d2h);
  if (e->side) cudaStreamDestroy(e->side);
  if (e->side2) cudaStreamDestroy(e->side2);
  delete e;
}

int32_t gwg_set_spectrum(gwg_engine* e, const double* basis, const double* lambda, int32_t where,
                         gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  return set_spectrum_impl(e, basis, e ? e->n : 0, lambda, where, st);
}

extern "C" int32_t gwg_internal_device_eig(double* a, int64_t n, int64_t lda, double* w,
                                           cudaStream_t stream, gwg_status* st);

int32_t gwg_set_kinship(gwg_engine* e, const double* phi, int32_t where, gwg_status* st) {
  NvtxRange nvtx_("gwg_set_kinship");
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  if (!phi) return set_status(st, GWG_DIMENSION, -1, -1, "null kinship matrix");
  e->have_spectrum = e->have_covariates = e->have_traits = false;
  if (int rc = upload_cols(e, e->basis, phi, e->n, e->n, where, e->comp, st)) return rc;
  GWG_CUDA_TRY(e->lambda.ensure(size_t(e->n) * sizeof(double)));
  if (int rc = gwg_internal_device_eig(e->basis.d(), e->n, e->np, e->lambda.d(), e->comp, st))
    return rc;
  if (int rc = spectrum_range(e, st)) return rc;
  invalidate_derived(e, true);
  e->have_spectrum = true;
  return GWG_OK;
}

int32_t gwg_set_covariates(gwg_engine* e, const double* xl, int32_t where, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  return set_covariates_impl(e, xl, e->n, where, false, st);
}

int32_t gwg_set_traits(gwg_engine* e, int64_t t, const double* y, const double* h2,
                       const double* sigma2, int32_t where, int32_t is_rotated, gwg_status* st) {
  NvtxRange nvtx_("gwg_set_traits");
  clear_status(st);
  if (int rc = check_engine(e, st, false)) return rc;
  return set_traits_impl(e, t, y, e->n, where, h2, sigma2, where, is_rotated != 0, st);
}

int32_t gwg_solve_snp_slab(gwg_engine* e, int64_t i0, int64_t mb, const double* x_r,
                           int32_t where, int32_t is_rotated, double* b_out, int32_t out_where,
                           int32_t layout, int64_t ldo, gwg_status* st) {
  NvtxRange nvtx_("gwg_solve_snp_slab");
  clear_status(st);
  if (int rc = check_engine(e, st, false)) return rc;
  if (!e->have_traits)
    return set_status(st, GWG_DIMENSION, -1, -1, "gwg_set_traits must come first");
  if (mb < 1 || i0 < 0 || !x_r || !b_out)
    return set_status(st, GWG_DIMENSION, -1, -1, "bad slab arguments (i0=%lld mb=%lld)",
                      (long long)i0, (long long)mb);
  if (mb > (int64_t(1) << 30))
    return set_status(st, GWG_DIMENSION, -1, -1, "slab too wide (mb=%lld)", (long long)mb);
  if (layout != GWG_LAYOUT_NUMPY && layout != GWG_LAYOUT_STREAM)
    return set_status(st, GWG_DIMENSION, -1, -1, "unknown layout %d", layout);
  if (layout == GWG_LAYOUT_STREAM && ldo < mb)
    return set_status(st, GWG_DIMENSION, -1, -1, "ldo (%lld) < mb (%lld)", (long long)ldo,
                      (long long)mb);
  const int64_t n = e->n, t = e->t, p = e->p;
  if (layout == GWG_LAYOUT_NUMPY) ldo = mb;
  // X' itself is only needed by the FP64 grid (the genotype split grid reads X'.X')
  if (is_rotated || !rotated_x_unused(e))
    GWG_CUDA_TRY(e->rot.ensure(size_t(e->np) * mb * sizeof(double)));
  GWG_CUDA_TRY(e->rot_sq.ensure(size_t(e->np) * mb * sizeof(double)));
  // before the rotation: it writes this slab's genotype verdict (word 2)
  if (int rc = begin_epoch(e, st)) return rc;
  e->i8_input = false;
  if (e->timings.size() <= e->timings_used) {
    gwg_engine::SlabTiming tm;
    for (cudaEvent_t& ev : tm.ev) GWG_CUDA_TRY(cudaEventCreate(&ev));
    e->timings.push_back(tm);
  }
  gwg_engine::SlabTiming& tmg = e->timings[e->timings_used++];
  tmg.joined = false;
  e->join_ev = tmg.ev + 7;
  e->join_timed = &tmg.joined;
  struct JoinEvReset {  // never left pointing into `timings` past this call
    gwg_engine* e;
    ~JoinEvReset() { e->join_ev = nullptr, e->join_timed = nullptr; }
  } join_ev_reset{e};
  if (int rc = mark_trait_fork(e, is_rotated, st)) return rc;
  GWG_CUDA_TRY(cudaEventRecord(tmg.ev[0], e->comp));
  if (is_rotated) {
    if (int rc = upload_cols(e, e->rot, x_r, n, mb, where, e->comp, st)) return rc;
    if (int rc = square_rotated(e, mb, st)) return rc;
  } else {
    const double* src = x_r;
    const bool direct = where == GWG_DEVICE && raw_ld(e) == n &&
                        (reinterpret_cast<uintptr_t>(x_r) & 15) == 0;
    if (!direct) {
      if (int rc = upload_cols(e, e->raw[0], x_r, n, mb, where, e->comp, st, raw_ld(e)))
        return rc;
      src = e->raw[0].d();
    }
    if (int rc = rotate_snps(e, src, raw_ld(e), mb, st)) return rc;
  }
  GWG_CUDA_TRY(cudaEventRecord(tmg.ev[1], e->comp));
  e->join_ev = nullptr;
  e->join_timed = nullptr;
  double* dev_out = b_out;
  if (out_where != GWG_DEVICE) {
    GWG_CUDA_TRY(e->out[0].ensure(size_t(mb) * t * p * sizeof(double)));
    dev_out = e->out[0].d();
  }
  const int64_t si = layout == GWG_LAYOUT_NUMPY ? t : 1;
  const int64_t sj = layout == GWG_LAYOUT_NUMPY ? 1 : (out_where == GWG_DEVICE ? ldo : mb);
  e->split_timed = false;
  GWG_CUDA_TRY(cudaEventRecord(tmg.ev[2], e->comp));
  e->split_ev = tmg.ev + 4;
  const int lrc = launch_slab(e, e->rot.d(), e->rot_sq.d(), mb, i0, kKeyStride, dev_out, si, sj, st);
  e->split_ev = nullptr;
  if (lrc) return lrc;
  tmg.split = e->split_timed;
  GWG_CUDA_TRY(cudaEventRecord(tmg.ev[3], e->comp));
  // a device output is asynchronous, like the device work that produces it:
  // the epoch stays open and its errors surface at the next synchronising call
  if (out_where == GWG_DEVICE) return GWG_OK;
  if (out_where != GWG_DEVICE) {
    if (layout == GWG_LAYOUT_NUMPY) {
      GWG_CUDA_TRY(cudaMemcpyAsync(b_out, dev_out, size_t(mb) * t * p * sizeof(double),
                                   cudaMemcpyDeviceToHost, e->comp));
    } else {
      GWG_CUDA_TRY(cudaMemcpy2DAsync(b_out, ldo * p * sizeof(double), dev_out,
                                     mb * p * sizeof(double), mb * p * sizeof(double), t,
                                     cudaMemcpyDeviceToHost, e->comp));
    }
    e->counters.bytes_stored += uint64_t(mb) * t * p * 8;
  }
  // Error coordinates are global: key = j * kKeyStride + (i0 + il).
  return end_epoch(e, st);
}

int32_t gwg_set_snp_coding(gwg_engine* e, int32_t coding, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  if (coding != GWG_SNP_REAL && coding != GWG_SNP_GENOTYPES && coding != GWG_SNP_AUTO)
    return set_status(st, GWG_DIMENSION, -1, -1, "unknown SNP coding %d", int(coding));
  if (coding == GWG_SNP_GENOTYPES && e->n >= kMaxGenotypeN)
    return set_status(st, GWG_DIMENSION, -1, -1,
                      "genotype coding needs n < 132,000 (exact int32 accumulation)");
  e->snp_coding = coding;
  return GWG_OK;
}

int32_t gwg_set_option(gwg_engine* e, int32_t option, int64_t value, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  auto flag = [&](bool& dst) -> int {
    if (value != 0 && value != 1)
      return set_status(st, GWG_DIMENSION, -1, -1, "option %d takes 0 or 1 (got %lld)",
                        int(option), (long long)value);
    dst = value != 0;
    return GWG_OK;
  };
  switch (option) {
    case GWG_OPT_SPLIT:
      return flag(e->split);
    case GWG_OPT_SBR_DIRECT: {
      bool direct = !e->lowrank;
      if (int rc = flag(direct)) return rc;
      if (direct == e->lowrank) invalidate_derived(e, false);  // E/F, W and D panels
      e->lowrank = !direct;
      return GWG_OK;
    }
    case GWG_OPT_REAL_SPLIT:
      return flag(e->real_split);
    case GWG_OPT_I8_CLUSTER:
      if (value < 0 || value > 5)
        return set_status(st, GWG_DIMENSION, -1, -1, "GWG_OPT_I8_CLUSTER takes 0..5 (got %lld)",
                          (long long)value);
      e->i8_cluster = int(value);
      return GWG_OK;
    case GWG_OPT_SBR_CFG:
      if (value < 0 || value >= gwg::kSbrConfigs)
        return set_status(st, GWG_DIMENSION, -1, -1, "GWG_OPT_SBR_CFG takes 0..%d (got %lld)",
                          gwg::kSbrConfigs - 1, (long long)value);
      if (int(value) != e->sbr_cfg) invalidate_derived(e, false);  // panel tiling changes
      e->sbr_cfg = int(value);
      e->sops = gwg::sbr_ops(e->sbr_cfg);
      return GWG_OK;
  }
  return set_status(st, GWG_DIMENSION, -1, -1, "unknown option %d", int(option));
}

int32_t gwg_get_option(gwg_engine* e, int32_t option, int64_t* value, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  if (!value) return set_status(st, GWG_DIMENSION, -1, -1, "null option value");
  switch (option) {
    case GWG_OPT_SPLIT: *value = e->split; return GWG_OK;
    case GWG_OPT_SBR_DIRECT: *value = !e->lowrank; return GWG_OK;
    case GWG_OPT_REAL_SPLIT: *value = e->real_split; return GWG_OK;
    case GWG_OPT_I8_CLUSTER: *value = e->i8_cluster; return GWG_OK;
    case GWG_OPT_SBR_CFG: *value = e->sbr_cfg; return GWG_OK;
  }
  return set_status(st, GWG_DIMENSION, -1, -1, "unknown option %d", int(option));
}

int32_t gwg_get_counters(gwg_engine* e, gwg_counters* out) {
  if (!e || !out) return GWG_DIMENSION;
  *out = e->counters;
  return GWG_OK;
}

void gwg_reset_counters(gwg_engine* e) {
  if (!e) return;
  e->counters = gwg_counters{};
  e->csum_cells = 0;
  e->timings_first = e->timings_used;  // queued solves belong to before the reset
  if (e->csum.ptr) {
    cudaSetDevice(e->device);
    cudaMemsetAsync(e->csum.ptr, 0, sizeof(unsigned long long), e->comp);
  }
}

int32_t gwg_synchronize(gwg_engine* e, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  GWG_CUDA_TRY(cudaStreamSynchronize(e->h2d));
  GWG_CUDA_TRY(cudaStreamSynchronize(e->d2h));
  // errors of asynchronous solves, and a trait failure queued by
  // gwg_set_traits, surface here at the latest
  if (e->epoch_open) return end_epoch(e, st);
  if (e->have_traits) return read_errors(e, st, false);
  GWG_CUDA_TRY(cudaStreamSynchronize(e->comp));
  return GWG_OK;
}

int64_t gwg_default_slab_snps(gwg_engine* e, int64_t m) {
  if (!e || e->t <= 0 || m <= 0) return 0;
  return default_slab(e, m);
}

void* gwg_compute_stream(gwg_engine* e) {
  if (!e) return nullptr;
  if (cudaSetDevice(e->device) == cudaSuccess) (void)join_side(e);  // side work ordered first
  return static_cast<void*>(e->comp);
}

}  // extern "C"
