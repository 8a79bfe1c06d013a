// engine_internal.cuh — engine state and host helpers shared by engine.cu
// (in-memory C ABI) and stream_io.cu (GWG1 file legs).  Not installed.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gwgrid_cuda.h"
#include "grid_split.cuh"
#include "kernel_table.cuh"
#include "linear_solve.cuh"

#define GWG_CUDA_TRY(expr)                                                                 \
  do {                                                                                     \
    cudaError_t err_ = (expr);                                                             \
    if (err_ != cudaSuccess)                                                               \
      return gwg_host::set_status(st, GWG_CUDA, -1, -1, "%s failed: %s (%s:%d)", #expr,    \
                                  cudaGetErrorString(err_), __FILE__, __LINE__);           \
  } while (0)

namespace gwg_host {

// NVTX range for profiler timelines (no-op unless a tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, need);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  double* d() const { return static_cast<double*>(ptr); }
};

// Page-locked host buffer kept by the engine across runs (cudaMallocHost is
// slow: the pipeline's staging buffers are allocated once and reused).
struct PinBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMallocHost(&ptr, need);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};


int set_status(gwg_status* st, int code, int64_t snp, int64_t trait, const char* fmt, ...);
void clear_status(gwg_status* st);
int64_t round_up(int64_t a, int64_t b);
int64_t ceil_div(int64_t a, int64_t b);
bool is_pinned_host(const void* p);

}  // namespace gwg_host

struct gwg_engine {
  int device = 0;
  int sms = 148;
  int64_t n = 0, p = 0, np = 0;
  gwg::KernelOps ops;
  gwg::LinOps lops;  // genotype split grid: per-p linear-solve kernel
  gwg::SbrOps sops;  // genotype split grid: S_BR kernel configuration
  cudaStream_t comp = nullptr, h2d = nullptr, d2h = nullptr;
  // trait-side operands of the split grid built concurrently with the SNP
  // side (mark_trait_fork / launch_split): side stream, fork and join events
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // helper stream of the split build (W's covariate columns beside its trait
  // column) and its fork / join events
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_traits_in = nullptr;  // gwg_set_traits' host uploads done
  cudaEvent_t ev_cov_fork = nullptr, ev_cov_join = nullptr;
  bool fork_pending = false;
  // trait-side device work queued on the side stream and not yet joined into
  // the compute stream (gwg_set_traits on the split path, then the split
  // build): join_side before anything on comp reads it
  bool side_pending = false;
  cudaEvent_t* join_ev = nullptr;  // the current slab's ev[7] (solve_snp_slab)
  bool* join_timed = nullptr;

  gwg_host::DevBuf basis, lambda, xl_raw, xl_rot;  // basis / xl_* / y_* / rot: leading dimension np
  bool have_spectrum = false, have_covariates = false;

  int64_t t = 0;
  bool have_traits = false;
  gwg_host::DevBuf y_raw, y_rot, h2, sigma2, bops, ctx;
  bool bops_valid = false;  // bops built for the current traits
  gwg::PrepArgs prep_args{};  // the last trait prep (rerun with panels on demand)

  gwg_host::DevBuf raw[2], rot, rot_sq, out[2], stage;  // rot / rot_sq: X' and X'.X', ld np
  gwg_host::DevBuf raw8[2];  // int8 genotype slabs (GWG_FORMAT_I8), n x rows, ld n
  gwg_host::DevBuf err;  // [0] trait error key, [1] cell error key, [2] genotype check
  // the run's SNP slabs came as int8 codes: a code outside [-127, 127] is an
  // error whatever the coding (err word 2)
  bool i8_input = false;
  // order-independent result checksum (gwg_run_options.checksum): [0] sum
  gwg_host::DevBuf csum;
  uint64_t csum_cells = 0;
  // pinned staging of the slab pipeline (pipeline.cu), reused across runs
  gwg_host::PinBuf pin_x[2];
  std::vector<gwg_host::PinBuf> pin_res;
  std::vector<cudaEvent_t> pipe_events;  // host-buffer hand-off events
  // SNP coding: 0 = real-valued (DMMA rotation), 1 = integer genotype codes
  // (exact int8 tcgen05 rotation); slices of Z are rebuilt after a new spectrum.
  int snp_coding = GWG_SNP_AUTO;
  bool slices_valid = false;
  gwg_host::DevBuf zslices, zscale, xi8;
  // Split grid for genotype slabs (grid_split.cuh): linear terms x_i^T W on
  // the int8 tensor cores fused with the solve, quadratic term S_BR on DMMA.
  // `split` = use it (GWG_OPT_SPLIT);
  // `slab_i8` = the current slab was rotated from integer codes (xi8 valid).
  bool split = true, slab_i8 = false;
  // GWG_SNP_AUTO: the current slab queued both paths, each gated on its
  // verdict (err word 2); gate_want = path of the launches being queued
  // (1 genotype, 0 FP64, -1 ungated)
  bool slab_auto = false;
  int gate_want = -1;
  // int8 kernels: 0 auto, 1 single CTAs, 2 CTA pairs multicasting B, 3 CTA
  // pairs multicasting the SNP tile (GWG_OPT_I8_CLUSTER)
  int i8_cluster = 0;
  int sbr_cfg = 0;  // GWG_OPT_SBR_CFG
  bool basis_t_valid = false, split_valid = false;
  gwg_host::DevBuf basis_t, vmat, wmat, wslices, wscale, dpanel, sbr;
  // S_BR = ((X'.X')^T E) F, the positive exponential-sum factorisation of D
  // (expsum.cpp): `sbr_terms` = r for the current traits, 0 = direct DMMA
  // contraction against D (inputs outside the factorisation's range, or
  // GWG_OPT_SBR_DIRECT = 1: `lowrank` = false).
  bool lowrank = true;
  int32_t sbr_terms = 0;
  bool expsum_valid = false;  // E, F (and sbr_terms) built for the current traits
  // FP64 path: S_BR from the factorised GEMMs and the grid kernel without the
  // D column (GWG_OPT_REAL_SPLIT = 0 keeps the fused S_BR)
  bool real_split = true;
  gwg_host::DevBuf epanel, fpanel, gmat, gpart, exps;
  gwg_host::DevBuf xepanel, umat, upart;  // upart: split-K partials of U  // W build through the factorisation: diag(X_L'_c) E, Z diag(X_L'_c) E
  // host copies of lambda / h2 / sigma2 when they were passed from the host:
  // the factorisation's range is then found without a device round trip
  std::vector<double> h2_host, s2_host;
  bool traits_host_valid = false;
  // device-resident traits: the range reduction is queued by gwg_set_traits
  // (pinned range_host, ev_range) and read when the split grid is built
  double* range_host = nullptr;
  cudaEvent_t ev_range = nullptr;
  bool range_pending = false;
  // min / max of the spectrum (found once per spectrum); lam_bad = non-finite
  double lam_lo = 0.0, lam_hi = 0.0;
  bool lam_bad = false;
  // the nodes on the device (exps + 8) were designed for this range
  double ex_lo = 0.0, ex_hi = -1.0, ex_lam0 = 0.0;
  int32_t ex_mult = 0, ex_r = 0;
  unsigned long long* err_host = nullptr;

  cudaEvent_t ev_h2d[2], ev_rot_done[2], ev_comp[2], ev_d2h_done[2];
  cudaEvent_t ev_k0, ev_k1, ev_r0, ev_r1;
  cudaEvent_t ev_wait = nullptr;    // gwg_wait_stream
  cudaEvent_t ev_signal = nullptr;  // gwg_signal_stream
  cudaEvent_t ev_s[3];     // split grid: before gls_sbr, before linear_solve, after it
  bool split_timed = false;
  // where launch_split records its three events (null: ev_s)
  cudaEvent_t* split_ev = nullptr;
  // Error epochs: the cell-error key (word 1) and the genotype verdict
  // (word 2) accumulate over every slab queued since the last synchronising
  // call; the first slab of an epoch resets them.  Asynchronous
  // device-output solves leave the epoch open (their errors surface at the
  // next gwg_synchronize / host-output solve / run_grid).
  bool epoch_open = false;
  // per-slab CUDA events of the open epoch's solves, turned into counters
  // when the epoch closes: [rotate begin, rotate end, grid begin, grid end,
  // sbr begin, linear begin, linear end]
  struct SlabTiming {
    // 0/1 around the SNP upload + rotation, 2/3 around the grid, 4/5/6 the
    // split grid's stages, 7/8 around the rotation's wait for the trait side
    // (split_build_ahead; not counted as rotation time)
    cudaEvent_t ev[9] = {};
    bool split = false;
    bool joined = false;
  };
  std::vector<SlabTiming> timings;
  size_t timings_used = 0;
  size_t timings_first = 0;  // pending timings before a counter reset are not counted
  std::vector<cudaEvent_t> slab_events;

  gwg_counters counters{};
};


namespace gwg_host {

// join = false (gwg_set_traits, gwg_solve_snp_slab): trait-side work queued
// on the side stream stays there; every other entry point joins it first
int check_engine(gwg_engine* e, gwg_status* st, bool join = true);
cudaError_t join_side(gwg_engine* e);
int split_build_ahead(gwg_engine* e, gwg_status* st);
int upload(gwg_engine* e, DevBuf& dst, const double* src, size_t count, int where,
           gwg_status* st);
int upload_cols(gwg_engine* e, DevBuf& dst, const double* src, int64_t lds, int64_t cols,
                int where, cudaStream_t s, gwg_status* st, int64_t ldd = 0);
int64_t raw_ld(const gwg_engine* e);
int rotate(gwg_engine* e, const double* src, int64_t cols, double* dst, gwg_status* st,
           int64_t lds = 0, double* dst_sq = nullptr, const double* basis = nullptr,
           int64_t ldd = 0);
// Split-grid trait operands (W slices, D panels) for the current traits.
int build_split(gwg_engine* e, gwg_status* st);
int mark_trait_fork(gwg_engine* e, bool rotated_input, gwg_status* st);
// Genotype split grid on raw slabs: X' is never materialised (only X'.X').
bool rotated_x_unused(const gwg_engine* e);
// exact int32 slice products need n * 127 * 128 < 2^31
constexpr int64_t kMaxGenotypeN = 132000;
// the path gate for the launches being queued (null = ungated)
inline const unsigned long long* gate_word(const gwg_engine* e) {
  return e->gate_want >= 0 ? static_cast<const unsigned long long*>(e->err.ptr) + 2 : nullptr;
}
int prepare_expsum(gwg_engine* e, gwg_status* st);
int sbr_gemm(gwg_engine* e, const double* a_op, int64_t kext, int64_t lda, int64_t rows,
             const double* panel, int64_t pk, int64_t cols, double* dst, int64_t ldd,
             bool rowmajor, gwg_status* st, int ksplit = 1, double* partials = nullptr,
             int64_t split_stride = 0, int64_t pad_chunks = 0);
int launch_sbr_stage(gwg_engine* e, const double* rot_sq, int64_t rows, int64_t ld_s,
                     gwg_status* st);
int launch_fused(gwg_engine* e, const double* rot, const double* rot_sq, int64_t rows, int64_t i0,
                 int64_t m_total, double* dev_out, int64_t out_si, int64_t out_sj,
                 gwg_status* st);
// Invalidate everything derived from traits / spectrum.
void invalidate_derived(gwg_engine* e, bool spectrum);
// SNP slab -> e->rot / e->rot_sq with the engine's SNP coding (DMMA or int8).
int rotate_snps(gwg_engine* e, const double* src, int64_t lds, int64_t cols, gwg_status* st);
// Copy the error words to the host (one sync) and report, in this order: a
// pending trait weight-floor failure (-1, j), an int8 code outside
// [-127, 127] (or, for GWG_SNP_GENOTYPES, a non-code value); cell errors are
// left to raise_cell_error.  slab_checks = false reports the trait word only
// (gwg_synchronize: the slab words belong to the call that queued the slab).
int read_errors(gwg_engine* e, gwg_status* st, bool slab_checks);
// Reset the per-slab words (cell key, genotype verdict); the trait word is
// reset by set_traits only.
int reset_errors(gwg_engine* e, gwg_status* st);
int launch_slab(gwg_engine* e, const double* rot, const double* rot_sq, int64_t rows, int64_t i0,
                int64_t m_total, double* dev_out, int64_t out_si, int64_t out_sj,
                gwg_status* st);
// Cell error keys are j * kKeyStride + i (global SNP index i < 2^34, trait
// j < 2^30): the minimum is the first failing cell in trait-major order
// whatever slabs, shards or calls produced it.
constexpr int64_t kKeyStride = int64_t(1) << 34;
int raise_cell_error(gwg_engine* e, gwg_status* st);
// Open an error epoch (reset the slab words) unless one is open.
int begin_epoch(gwg_engine* e, gwg_status* st);
// Close it: wait for the compute stream, fold pending slab timings into the
// counters, report (trait, genotype, cell) errors in that order.
int end_epoch(gwg_engine* e, gwg_status* st);
// rot_sq <- rot .* rot for `cols` already-rotated columns
int square_rotated(gwg_engine* e, int64_t cols, gwg_status* st);
int64_t default_slab(const gwg_engine* e, int64_t m);

// The slab pipeline (pipeline.cu), run_grid's traversal on the device.
// Input: slab s arrives either straight from a pinned host array (x_direct,
// column-major, ld n, element size by format) or through read_fn, which
// fills a pinned n x rows staging slab (ld n) on a reader thread.  Output:
// either straight into a pinned host array (b_direct; NUMPY rows at
// il * t * p, STREAM at (j * ldb + il) * p) or through write_fn, which drains
// a pinned slab-local result buffer (NUMPY (il*t + j)*p, STREAM
// (j*rows + il)*p) on a writer thread.  i0 arguments of the callbacks are
// local to the run (0 = x's first column).
using SlabRead = std::function<bool(int64_t i0, int64_t rows, void* dst)>;
using SlabWrite = std::function<bool(int64_t i0, int64_t rows, const double* src)>;
struct PipeSpec {
  int64_t m = 0;         // SNP columns of this run
  int64_t i0 = 0;        // global SNP index of its first column
  int64_t mb = 0;        // slab width
  int fmt = GWG_FORMAT_F64;
  bool rotated = false;  // f64 slabs already rotated (the FP64 path)
  int layout = GWG_LAYOUT_NUMPY;
  bool dbuf = true;
  int ring = 2;          // pinned result buffers behind write_fn
  bool checksum = false;
  const void* x_direct = nullptr;
  SlabRead read_fn;
  double* b_direct = nullptr;
  int64_t ldb = 0;       // STREAM layout row length of b_direct (cells)
  SlabWrite write_fn;
};
struct PipeStats {
  uint64_t loaded = 0, stored = 0;
  double stall_ms = 0.0;
  int io_error = 0;      // 1 = read_fn failed, 2 = write_fn failed
};
int run_pipeline(gwg_engine* e, const PipeSpec& spec, PipeStats* stats, gwg_status* st);
// gwg_run_grid's argument checks and spec (shared with the device group)
int run_grid_impl(gwg_engine* e, int64_t m, const void* x_r_host, double* b_host,
                  const gwg_run_options* opts, gwg_counters* counters, gwg_status* st);
// memcpy over a few threads (pageable user memory <-> pinned staging)
void parallel_copy(void* dst, const void* src, size_t bytes);
// Shared-operand installs with explicit leading dimensions and locations (the
// device group broadcasts device-resident, already rotated operands).
int set_spectrum_impl(gwg_engine* e, const double* basis, int64_t ldb, const double* lambda,
                      int where, gwg_status* st);
int set_covariates_impl(gwg_engine* e, const double* xl, int64_t ldx, int where, bool rotated,
                        gwg_status* st);
int set_traits_impl(gwg_engine* e, int64_t t, const double* y, int64_t ldy, int y_where,
                    const double* h2, const double* sigma2, int s_where, bool rotated,
                    gwg_status* st);
// int8 genotype slab (n x cols, ld n) -> e->rot_sq (and xi8) with the engine's coding
int rotate_snps_i8(gwg_engine* e, const int8_t* src, int64_t cols, gwg_status* st);
// accumulate the result checksum of one slab-local result buffer
int launch_checksum(gwg_engine* e, const double* out, int64_t rows, int layout, int64_t i0,
                    gwg_status* st);

}  // namespace gwg_host
