/*
 * gwgrid_cuda.h — C ABI of the B200-native GLS-grid engine (the drop-in
 * boundary for the reference gwgrid hot path).
 *
 * The reference (gwgrid, arXiv 1210.7683) has no plugin/FFI layer; its seam
 * for this path is the C++ library API in proj/include/gwgrid/grid.hpp, called
 * from run_grid's compute phase (proj/src/grid.cpp:541-552), plus the in-memory
 * Python contract gwgrid.solve_grid (proj/python/bindings.cpp:115-190,318-328).
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes, column-major FP64 operands, int64 dimensions.
 *   - Every call returns a status code (0 = ok) and fills *st when non-null.
 *   - Codes map 1:1 onto the reference error hierarchy
 *     (proj/include/gwgrid/types.hpp:34-94); GWG_NOT_POSITIVE_DEFINITE carries
 *     the grid coordinates (snp_index, trait_index), -1 = not applicable.
 *   - One engine per device; calls on one engine must be serialised by the
 *     caller (the reference's CT coordinator thread, grid.cpp:519-552).
 *   - `where` flags say whether a pointer is host (GWG_HOST) or device
 *     (GWG_DEVICE) memory.  Host buffers may be pageable or pinned; pinned
 *     buffers give overlapped transfers.
 *   - Output layouts: GWG_LAYOUT_NUMPY writes cell (i, j) at (i*t + j)*p
 *     (the numpy (m, t, p) array of bindings.cpp:176-184); GWG_LAYOUT_STREAM
 *     writes it at (j*m + i)*p (the GWG1 result stream, stream.hpp:31-34).
 */
#ifndef GWGRID_CUDA_H_
#define GWGRID_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum gwg_code {
  GWG_OK = 0,
  GWG_DIMENSION = 1,               /* DimensionError          types.hpp:38-40 */
  GWG_NON_SYMMETRIC = 2,           /* NonSymmetricError       types.hpp:43-45 */
  GWG_BACKEND = 3,                 /* BackendError            types.hpp:48-50 */
  GWG_NOT_POSITIVE_DEFINITE = 4,   /* NotPositiveDefiniteError types.hpp:55-63 */
  GWG_IO = 5,                      /* IoError                 types.hpp:66-68 */
  GWG_INFEASIBLE_BUDGET = 6,       /* InfeasibleBudgetError   types.hpp:91-93 */
  GWG_CUDA = 7                     /* device/runtime failure (no reference analogue) */
};

enum gwg_where { GWG_HOST = 0, GWG_DEVICE = 1 };
enum gwg_layout { GWG_LAYOUT_NUMPY = 0, GWG_LAYOUT_STREAM = 1 };
enum gwg_snp_coding { GWG_SNP_REAL = 0, GWG_SNP_GENOTYPES = 1, GWG_SNP_AUTO = 2 };

typedef struct gwg_status {
  int32_t code;
  int64_t snp_index;
  int64_t trait_index;
  char msg[256];
} gwg_status;

/* Analytic counters, same buckets as RunCounters (counters.hpp:62-127), plus
 * device-side timings. */
typedef struct gwg_counters {
  uint64_t preloop_flops;      /* rotations of X_L and X_R (2 n^2 cols)            */
  uint64_t loop_flops;         /* trait contexts + cells, reference convention      */
  uint64_t grid_flops;         /* 2 n (p+1) per cell: the DMMA contraction work     */
  uint64_t bytes_loaded;       /* host->device bytes                                 */
  uint64_t bytes_stored;       /* device->host bytes                                 */
  uint64_t context_builds;     /* trait-prep launches (one per gwg_set_traits)       */
  uint64_t kernel_launches;    /* launches of this library's own kernels            */
  double grid_kernel_ms;       /* summed CUDA-event time of the grid launches        */
  double rotate_ms;            /* summed CUDA-event time of the SNP rotations        */
  double wall_ms;              /* host wall time of the last run_grid                */
  /* genotype split grid (gwg_solve_snp_slab only), both inside grid_kernel_ms:
   * linear_ms = int8 linear terms + Cholesky solve (linear_solve_kernel),
   * quad_ms = S_BR on DMMA (gls_sbr_kernel launches) */
  double linear_ms;
  double quad_ms;
  /* S_BR work actually issued on DMMA: 2 n t per SNP direct, 2 r (n + t) per
   * SNP factorised; sbr_terms = r of the last slab (0 = direct contraction) */
  uint64_t sbr_flops;
  int64_t sbr_terms;
  /* run_grid: compute-side waits on slab I/O (pipeline_run's stall,
   * pipeline.hpp:106-136): gaps of the compute stream between slabs (first
   * H2D included) plus the tail of result stores after the last slab */
  double io_stall_ms;
  /* order-independent checksum of every b_ij solved with
   * gwg_run_options.checksum = 1 since the last reset: the wrapping sum over
   * cells and components of gwg_cell_hash(i, j, c, bits(b_ijc)) — identical
   * for any slab width, layout, shard split or GPU count */
  uint64_t checksum;
  uint64_t checksum_cells;
} gwg_counters;

/* Input formats of SNP slabs given to gwg_run_grid. */
enum gwg_snp_format {
  GWG_FORMAT_F64 = 0,  /* x_r is double (any real values; raw or rotated)          */
  GWG_FORMAT_I8 = 1    /* x_r is int8_t genotype codes in [-127, 127], 1 byte each:
                          8x less host memory and PCIe traffic; the genotype path
                          runs on them directly (GWG_SNP_REAL converts to FP64 on
                          the device); -128 is a GWG_DIMENSION error */
};

/* Result sink: receives each slab's cells from a pinned host buffer that is
 * valid only during the call: rows SNPs starting at global SNP index i0
 * against all t traits, in the run's layout, slab-local
 * (NUMPY: (il*t + j)*p; STREAM: (j*rows + il)*p).  Called from one writer
 * thread per engine, in slab order; gwg_group_run_grid calls it from several
 * threads at once (one per device).  A non-zero return aborts the run with
 * GWG_IO. */
typedef int32_t (*gwg_result_sink)(void* user, int64_t i0, int64_t rows, const double* cells);

typedef struct gwg_run_options {
  int64_t mb;          /* SNP columns per streamed slab; 0 = engine default       */
  int32_t layout;      /* gwg_layout of the host result buffer                    */
  int32_t double_buffer; /* 1 = overlap H2D / compute / D2H (default)            */
  int32_t snp_format;  /* gwg_snp_format of x_r (default GWG_FORMAT_F64)         */
  int32_t checksum;    /* 1 = accumulate the device checksum into counters        */
  int64_t i0;          /* global SNP index of x_r's first column (a shard of a
                          larger grid): error coordinates and checksum keys are
                          global; results still start at b[0]                    */
  int64_t ldb;         /* STREAM layout: cells per trait row of b (>= m; 0 = m)  */
  gwg_result_sink sink; /* non-NULL: results leave through the sink (rotating
                          pinned buffers; b_host unused and may be NULL)        */
  void* sink_user;
  int32_t ring;        /* pinned result buffers rotated through the sink (0 = 2) */
  int32_t reserved;
} gwg_run_options;

typedef struct gwg_engine gwg_engine;

/* Library identity: "gwgrid_cuda <version> sm_100a". */
const char* gwg_version(void);

/* Create an engine on `device` for n samples and p predictors per fit
 * (p-1 shared covariates + 1 variant column).  Replaces the construction of
 * GridPrecompute (grid.hpp:81-87).  Returns NULL and fills *st on failure. */
gwg_engine* gwg_engine_create(int32_t device, int64_t n, int64_t p, gwg_status* st);
void gwg_engine_destroy(gwg_engine* e);

/* Install the kinship eigensystem Phi = Z diag(lambda) Z^T (Z: n x n col-major,
 * lambda ascending).  The eigendecomposition itself stays on the CPU
 * (eigendecompose_kinship, gls.cpp:16-46); this replaces its storage in
 * GridPrecompute::spectrum (grid.hpp:81-87). */
int32_t gwg_set_spectrum(gwg_engine* e, const double* basis, const double* lambda,
                         int32_t where, gwg_status* st);

/* Device eigendecomposition of the kinship matrix with the reference's
 * contract (eigendecompose_kinship, gls.cpp:16-46): symmetry gate
 * max|Phi-Phi^T| <= 1e-12 max|Phi| (else GWG_NON_SYMMETRIC), ascending
 * eigenvalues, each eigenvector's largest-magnitude entry made positive.
 * Standalone (no engine): phi n x n col-major on `where`; basis (n x n) and
 * values (n) written to `out_where`. */
int32_t gwg_eigendecompose(int32_t device, int64_t n, const double* phi, int32_t where,
                           double* basis, double* values, int32_t out_where, gwg_status* st);

/* precompute_grid's eigendecomposition on the device (grid.cpp:83-101): the
 * engine eigendecomposes phi (n x n) in place and installs the spectrum, so
 * the basis never travels to the host.  Alternative to gwg_set_spectrum. */
int32_t gwg_set_kinship(gwg_engine* e, const double* phi, int32_t where, gwg_status* st);

/* Install X_L (n x (p-1), col-major, raw) and rotate it on the device:
 * X_L' = Z^T X_L.  Replaces rotate_columns(Z, X_L) inside precompute_grid
 * (grid.cpp:83-101). */
int32_t gwg_set_covariates(gwg_engine* e, const double* xl, int32_t where, gwg_status* st);

/* Install t traits Y (n x t col-major; raw unless is_rotated) with per-trait
 * h2[t], sigma2[t]; rotates Y on the device and builds every trait context
 * (weights d, D = 1/d, D.Y', D.X_L', S_TL, chol(S_TL), z_T) in one kernel.
 * Replaces transform_trait_slab + build_trait_contexts (grid.cpp:135-175) and
 * the per-pass load_pass (grid.cpp:501-517).  Asynchronous: the call queues
 * its work and returns without a host round trip — on the genotype split path
 * on the engine's side stream, so it runs under the next slab's upload and
 * code conversion; the compute stream is ordered after it before anything
 * reads it (and by gwg_compute_stream, gwg_signal_stream, gwg_synchronize).
 * Device operands are read asynchronously: keep them unchanged until the next
 * synchronising call.  A trait whose rotated
 * weights fail the relative floor (gls.cpp:59-75) is reported as
 * GWG_NOT_POSITIVE_DEFINITE, snp_index = -1, trait_index = the first such j,
 * by the next call that synchronises (gwg_solve_snp_slab, gwg_run_grid*,
 * gwg_synchronize), ahead of any cell error. */
int32_t gwg_set_traits(gwg_engine* e, int64_t t, const double* y, const double* h2,
                       const double* sigma2, int32_t where, int32_t is_rotated,
                       gwg_status* st);

/* Solve the cells of one SNP slab against every installed trait (with a
 * device b_out the call is asynchronous: it returns once the work is queued
 * on the engine's compute stream, and errors — a failing cell with its
 * coordinates, a trait failure, non-code genotypes — are reported by the next
 * synchronising call: gwg_synchronize, a host-output solve or gwg_run_grid):
 * rows = mb SNP columns starting at global SNP index i0, x_r = n x mb
 * col-major (raw unless is_rotated; rotated on the device when raw).
 * Results for cell (il, j) go to b_out at
 *   layout NUMPY : (il * t + j) * p           (slab-local numpy order)
 *   layout STREAM: (j * ldo + il) * p         (result-stream order, ldo >= mb)
 * b_out may be host or device memory (out_where).  Replaces
 * transform_snp_slab + compute_tile (grid.cpp:125-133, 220-273); the first
 * failing cell in trait-major order (j*m_total + i) is reported with its
 * global coordinates like compute_block (grid.cpp:206-212). */
int32_t gwg_solve_snp_slab(gwg_engine* e, int64_t i0, int64_t mb, const double* x_r,
                           int32_t where, int32_t is_rotated, double* b_out,
                           int32_t out_where, int32_t layout, int64_t ldo,
                           gwg_status* st);

/* Stream the whole m x t grid from host memory: X_R (n x m, raw unless
 * rotated, col-major; double or int8 codes per opts->snp_format) in
 * mb-column slabs through double-buffered H2D / rotate+grid / D2H on three
 * CUDA streams, into the host result buffer b (m*t*p doubles, `layout`) or
 * through opts->sink.  Replaces preloop_stream_transform + run_grid
 * (grid.cpp:378-641) with its double-buffered pipeline_run
 * (pipeline.hpp:78-137) for in-memory operands; counters->io_stall_ms is
 * pipeline_run's stall. */
int32_t gwg_run_grid(gwg_engine* e, int64_t m, const void* x_r_host, double* b_host,
                     const gwg_run_options* opts, gwg_counters* counters,
                     gwg_status* st);

/* The per-(cell, component) term of the order-independent result checksum
 * (host copy of the device formula, for checking a downloaded grid):
 * a splitmix64 mix of the global SNP index i, trait index j, component c and
 * the IEEE-754 bits of b_ijc.  The checksum is the wrapping uint64 sum of
 * these terms over every component of every cell. */
uint64_t gwg_cell_hash(int64_t i, int64_t j, int64_t c, uint64_t bits);

/* Order the engine's compute stream after all work already queued on
 * `stream` (a cudaStream_t as void*, e.g. torch's current stream), without a
 * host round trip: device operands produced there are then safe to read. */
int32_t gwg_wait_stream(gwg_engine* e, void* stream, gwg_status* st);

/* The converse: order `stream` after all work queued on the engine so far
 * (device event, no host round trip) — e.g. torch's current stream before it
 * reads a device output of an asynchronous gwg_solve_snp_slab. */
int32_t gwg_signal_stream(gwg_engine* e, void* stream, gwg_status* st);

/* ---- One process, several GPUs --------------------------------
 * A group holds one engine per listed device (a device may repeat).  The
 * shared operands go host -> the first device once and are then broadcast
 * device-to-device (peer copies over NVLink / NVSwitch): the spectrum, the
 * rotated covariates X_L' and the rotated traits Y' (plus h2, sigma2); each
 * device builds its own trait contexts.  gwg_group_run_grid shards m into
 * contiguous, balanced column ranges, one per device, and runs gwg_run_grid
 * on each from its own host thread with its own pinned buffers; there is no
 * other collective.  Results land in the caller's buffer (or sink) at global
 * positions; counters are summed (checksum included: it does not depend on
 * the split); the first failing cell in trait-major order over the whole grid
 * is reported, like the one-device run.  Replaces run_grid's worker
 * parallelism (grid.cpp:519-639) at device granularity. */
typedef struct gwg_group gwg_group;
gwg_group* gwg_group_create(const int32_t* devices, int32_t count, int64_t n, int64_t p,
                            gwg_status* st);
void gwg_group_destroy(gwg_group* g);
int32_t gwg_group_size(const gwg_group* g);
/* The k-th device's engine (options, counters, single-device calls). */
gwg_engine* gwg_group_engine(gwg_group* g, int32_t k);
int32_t gwg_group_set_spectrum(gwg_group* g, const double* basis, const double* lambda,
                               int32_t where, gwg_status* st);
int32_t gwg_group_set_covariates(gwg_group* g, const double* xl, int32_t where,
                                 gwg_status* st);
int32_t gwg_group_set_traits(gwg_group* g, int64_t t, const double* y, const double* h2,
                             const double* sigma2, int32_t where, int32_t is_rotated,
                             gwg_status* st);
int32_t gwg_group_set_snp_coding(gwg_group* g, int32_t coding, gwg_status* st);
int32_t gwg_group_set_option(gwg_group* g, int32_t option, int64_t value, gwg_status* st);
/* Shard k covers SNP columns [bounds[k], bounds[k+1]) of an m-column run
 * (bounds has size() + 1 entries). */
int32_t gwg_group_shards(const gwg_group* g, int64_t m, int64_t* bounds);
int32_t gwg_group_run_grid(gwg_group* g, int64_t m, const void* x_r_host, double* b_host,
                           const gwg_run_options* opts, gwg_counters* counters,
                           gwg_status* st);

/* Independent verification route (CholeskyOracle, gls.cpp:188-244, as used by
 * gwgrid.verify_grid, bindings.cpp:192-222): for every trait j, factor
 * M_j = sigma2_j (h2_j Phi + (1 - h2_j) I) on the device, solve the GLS of
 * every cell through L^-1 [X_L | y_j | x_i] and the p x p normal equations,
 * and return the max norm-wise relative error |b - ref| / |ref| of b
 * ((m, t, p) numpy order, host) in *max_rel_err, and every cell's error in
 * cell_err ((m, t) numpy order) when non-null.  All operands raw, host,
 * column-major (kinship n x n, xl n x (p-1), snps n x m, traits n x t). */
int32_t gwg_verify_grid(int32_t device, int64_t n, int64_t p, int64_t m, int64_t t,
                        const double* kinship, const double* xl, const double* snps,
                        const double* traits, const double* h2, const double* sigma2,
                        const double* b, double* cell_err, double* max_rel_err,
                        gwg_status* st);

/* ---- GWG1 file legs (proj/include/gwgrid/stream.hpp:15-41) ----------------
 * 64-byte little-endian header: "GWG1", u16 version 1, u8 kind (1 snp, 2 trait,
 * 3 result, 4 operand), u8 element type 0 (f64), u64 dims[3], u8 layout 0,
 * u8 completeness (0 = complete), zero padding; column-major f64 payload;
 * result cell (i, j) at element (j*m + i)*p.  Readers validate magic,
 * version, kind, element type, layout, completeness and exact file length
 * like InputStream::open (stream.cpp:219-257); failures are GWG_IO. */

/* Header of a GWG1 file: kind, dims[3], complete flag (no payload checks). */
int32_t gwg_stream_info(const char* path, int32_t* kind, int64_t* dims, int32_t* complete,
                        gwg_status* st);

/* load_pass from a trait stream (kind 2: n x t columns, then h2[t], sigma2[t]);
 * equivalent to gwg_set_traits on the file's payload. */
int32_t gwg_set_traits_file(gwg_engine* e, const char* traits_path, gwg_status* st);

/* run_grid over GWG1 files (grid.cpp:454-641): the SNP stream (kind 1, raw, or
 * rotated when snps_rotated) is read slab by slab by a reader thread into
 * pinned buffers, solved on the device, and a writer thread stores each slab's
 * cells into the result stream out_path (kind 3, dims (m, t, p)).  The output
 * is created incomplete and finalized only when every cell landed and none
 * failed; a failing cell returns GWG_NOT_POSITIVE_DEFINITE and leaves the file
 * unreadable, like the reference. */
int32_t gwg_run_grid_files(gwg_engine* e, const char* snps_path, int32_t snps_rotated,
                           const char* out_path, const gwg_run_options* opts,
                           gwg_counters* counters, gwg_status* st);

/* How SNP slabs are coded (no reference counterpart: the reference stores
 * X_R as doubles and its generator draws genotype codes, datagen.cpp /
 * BASELINE.json).  GWG_SNP_REAL: any real values; the rotation and the grid
 * run on the FP64 tensor pipe (DMMA).  GWG_SNP_GENOTYPES: every SNP value is
 * an integer code in [-127, 127] (e.g. genotypes 0/1/2), checked on the
 * device (violations fail with GWG_DIMENSION); n < 132,000.  Then the
 * rotation X'.X' and the p linear terms of every cell (x^T W, W = Z D [X_L' Y'])
 * run exactly on the int8 tensor cores (tcgen05.mma kind::i8, seven 8-bit
 * slices, exact int64 recombination, one rounding) and only S_BR = (X'.X')^T D
 * stays on DMMA, factorised as ((X'.X')^T E) F through a positive exponential
 * sum of D (gwg_exp_sum_design; GWG_OPT_SBR_DIRECT = 1 forces the direct
 * contraction) — the same cells to rounding
 * (~1e-14 norm-wise), ~6.5x faster than the all-FP64 path at BASELINE config
 * 1; results stay bitwise independent of slab geometry.  GWG_SNP_AUTO (the
 * default): per slab, the device check decides — a slab of codes takes the
 * genotype path, any other slab the FP64 path (both are queued; the kernels
 * of the path not taken return at once, no host round trip), never an error.
 * Pre-rotated slabs (is_rotated = 1) always take the FP64 path. */
int32_t gwg_set_snp_coding(gwg_engine* e, int32_t coding, gwg_status* st);

/* Engine options (no reference counterpart: they select among this library's
 * own kernel schedules).  Every choice gives the reference's cells to
 * rounding, and the result is a pure function of the inputs and the options
 * (never of the caller's environment or the slab geometry).
 *   GWG_OPT_SPLIT       1 (default): genotype slabs take the split grid
 *                       (S_BR on DMMA, exact int8 linear terms + solve);
 *                       0: the all-FP64 fused grid kernel for them too.
 *   GWG_OPT_SBR_DIRECT  0 (default): S_BR through the positive exponential-sum
 *                       factorisation of D where it applies; 1: always the
 *                       direct contraction (X'.X')^T D.
 *   GWG_OPT_REAL_SPLIT  1 (default): the FP64 path with t >= 256 takes the
 *                       factorised S_BR and the grid kernel without the D
 *                       column; 0: the single fused kernel.
 *   GWG_OPT_I8_CLUSTER  0 (default, auto), 1 single CTAs, 2 CTA pairs
 *                       multicasting the W/Z-slice tile, 3 CTA pairs
 *                       multicasting the SNP tile, 4 CTA pairs running one
 *                       cta_group::2 MMA with half of the slice tile each
 *                       (32-row tiles; else 2), 5 2 x 2 clusters multicasting
 *                       halves of both operands (linear terms; the rotation
 *                       takes 2) — all bitwise identical.
 *   GWG_OPT_SBR_CFG     gls_sbr_kernel tile configuration index (default 0). */
enum gwg_option {
  GWG_OPT_SPLIT = 1,
  GWG_OPT_SBR_DIRECT = 2,
  GWG_OPT_REAL_SPLIT = 3,
  GWG_OPT_I8_CLUSTER = 4,
  GWG_OPT_SBR_CFG = 5
};
int32_t gwg_set_option(gwg_engine* e, int32_t option, int64_t value, gwg_status* st);
int32_t gwg_get_option(gwg_engine* e, int32_t option, int64_t* value, gwg_status* st);

/* Counters accumulated since the last reset. */
int32_t gwg_get_counters(gwg_engine* e, gwg_counters* out);
void gwg_reset_counters(gwg_engine* e);

/* Wait for all work queued by this engine. */
int32_t gwg_synchronize(gwg_engine* e, gwg_status* st);

/* The engine's compute stream (cudaStream_t as void*), so callers can order
 * their own device work (timing events, torch streams) against it; work still
 * queued on the engine's side stream (gwg_set_traits) is joined into it first. */
void* gwg_compute_stream(gwg_engine* e);

/* The SNP-slab width gwg_run_grid / gwg_run_grid_files use for an m-column run
 * when gwg_run_options.mb is 0, for the traits currently installed (whole
 * tile waves near a 96 MB result slab): the resolved `mb` that the reference's
 * solve report prints (TileParams::resolved, grid.cpp:37-62).  0 if no traits
 * are installed. */
int64_t gwg_default_slab_snps(gwg_engine* e, int64_t m);

/* Positive exponential sum for 1/x on [x_min, x_max] (the low-rank
 * factorisation of the GLS weights behind the genotype grid's S_BR term, see
 * csrc/expsum.cpp):  1/x ~= sum_r w[r] exp(-s[r] x),  s[0] = 0, all w > 0,
 * relative error <= ~2^-52 uniformly.  *terms = r, a multiple of `multiple`;
 * s / w may be NULL to query r.  GWG_DIMENSION if x_min <= 0, x_max < x_min,
 * or r would exceed max_terms.  Host-only (no device needed). */
int32_t gwg_exp_sum_design(double x_min, double x_max, int32_t multiple, int32_t max_terms,
                           double* s, double* w, int32_t* terms);

/* Seeded synthetic inputs with BASELINE.json's generators (counter-based
 * splitmix64 per (seed, matrix, column, row), so any column range is
 * reproducible independently).  matrix ids: 1 = kinship genotypes G,
 * 2 = covariates, 3 = SNPs X_R, 4 = traits Y, 5 = h2.  Host-side, threaded. */
void gwg_gen_genotypes(uint64_t seed, int32_t matrix, int64_t rows, int64_t col0,
                       int64_t ncols, int32_t standardize, double* out, int64_t ld);
void gwg_gen_normals(uint64_t seed, int32_t matrix, int64_t rows, int64_t col0,
                     int64_t ncols, double* out, int64_t ld);
void gwg_gen_uniform(uint64_t seed, int32_t matrix, int64_t count, double lo, double hi,
                     double* out);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* GWGRID_CUDA_H_ */
