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
} gwg_counters;

typedef struct gwg_run_options {
  int64_t mb;          /* SNP columns per streamed slab; 0 = engine default       */
  int32_t layout;      /* gwg_layout of the host result buffer                    */
  int32_t double_buffer; /* 1 = overlap H2D / compute / D2H (default)            */
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
 * the per-pass load_pass (grid.cpp:501-517).  A trait whose rotated weights
 * fail the relative floor (gls.cpp:59-75) fails with
 * GWG_NOT_POSITIVE_DEFINITE, snp_index = -1, trait_index = the first such j. */
int32_t gwg_set_traits(gwg_engine* e, int64_t t, const double* y, const double* h2,
                       const double* sigma2, int32_t where, int32_t is_rotated,
                       gwg_status* st);

/* Solve the cells of one SNP slab against every installed trait:
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

/* Stream the whole m x t grid from host memory: X_R (n x m, raw, col-major)
 * in mb-column slabs through double-buffered H2D / rotate+grid / D2H on three
 * CUDA streams, into the host result buffer b (m*t*p doubles, `layout`).
 * Replaces preloop_stream_transform + run_grid (grid.cpp:378-641) for
 * in-memory operands (the GWG1 file legs are out of scope). */
int32_t gwg_run_grid(gwg_engine* e, int64_t m, const double* x_r_host, double* b_host,
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
 * sum of D (gwg_exp_sum_design; GWG_SNP_GENOTYPES with GWG_SBR_DIRECT=1 in the
 * environment forces the direct contraction) — the same cells to rounding
 * (~1e-14 norm-wise), ~6.5x faster than the all-FP64 path at BASELINE config
 * 1; results stay bitwise independent of slab geometry.  GWG_SNP_AUTO (the
 * default): per slab, the device check decides — a slab of codes takes the
 * genotype path, any other slab the FP64 path (both are queued; the kernels
 * of the path not taken return at once, no host round trip), never an error.
 * Pre-rotated slabs (is_rotated = 1) always take the FP64 path. */
int32_t gwg_set_snp_coding(gwg_engine* e, int32_t coding, gwg_status* st);

/* Counters accumulated since the last reset. */
int32_t gwg_get_counters(gwg_engine* e, gwg_counters* out);
void gwg_reset_counters(gwg_engine* e);

/* Wait for all work queued by this engine. */
int32_t gwg_synchronize(gwg_engine* e, gwg_status* st);

/* The engine's compute stream (cudaStream_t as void*), so callers can order
 * their own device work (timing events, torch streams) against it. */
void* gwg_compute_stream(gwg_engine* e);

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
