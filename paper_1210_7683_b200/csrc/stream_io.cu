// stream_io.cu — GWG1 file legs of the engine (a9/a10/a12).
//
// The reference streams the grid out of core through GWG1 files
// (proj/include/gwgrid/stream.hpp:15-41, proj/src/stream.cpp): 64-byte
// little-endian header (magic "GWG1", version 1, kind 1 snp / 2 trait /
// 3 result / 4 operand, element type 0 = f64, dims x3, layout 0, completeness
// byte 33), column-major payload, result cell (i, j) at (j*m + i)*p.  Outputs
// are created incomplete and finalized only after every cell landed, so
// interrupted or failed runs leave files readers reject.
//
// Here the traversal of run_grid (grid.cpp:454-641) becomes:
//   reader thread  : pread SNP slab s into pinned host buffer hx[s%2]
//   coordinator    : H2D -> (rotate) -> fused grid -> D2H on three CUDA streams
//   writer thread  : pwrite the t contiguous cell runs of slab s from pinned hb[s%2]
// the same two-agent double-buffer discipline as IoAgent/pipeline_run
// (pipeline.hpp:16-137), with CUDA events as the ownership hand-off.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine_internal.cuh"

using namespace gwg_host;

namespace {

constexpr size_t kHeader = 64;

struct Header {
  uint8_t kind = 0;
  uint64_t dims[3] = {0, 0, 0};
  bool complete = false;
};

uint64_t payload_bytes(const Header& h) {
  switch (h.kind) {
    case 1:
    case 4:
      return h.dims[0] * h.dims[1] * 8;
    case 2:
      return h.dims[1] * (h.dims[0] + 2) * 8;
    case 3:
      return h.dims[0] * h.dims[1] * h.dims[2] * 8;
  }
  return 0;
}

void encode(const Header& h, unsigned char* b) {
  std::memset(b, 0, kHeader);
  b[0] = 'G';
  b[1] = 'W';
  b[2] = 'G';
  b[3] = '1';
  b[4] = 1;  // version, little endian u16
  b[5] = 0;
  b[6] = h.kind;
  b[7] = 0;  // float64
  for (int d = 0; d < 3; ++d)
    for (int q = 0; q < 8; ++q) b[8 + 8 * d + q] = static_cast<unsigned char>(h.dims[d] >> (8 * q));
  b[32] = 0;  // column-major slabs
  b[33] = h.complete ? 0 : 1;
}

const char* kind_name(int k) {
  switch (k) {
    case 1: return "variant stream";
    case 2: return "trait stream";
    case 3: return "result grid";
    case 4: return "operand matrix";
  }
  return "?";
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// Positional I/O that retries interrupted calls and short transfers, like
// the reference's read_exact / write_exact (proj/src/stream.cpp:47-81).
bool pread_all(int fd, void* dst, size_t bytes, uint64_t off) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, bytes, off_t(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    p += r;
    bytes -= size_t(r);
    off += uint64_t(r);
  }
  return true;
}

bool pwrite_all(int fd, const void* src, size_t bytes, uint64_t off) {
  const char* p = static_cast<const char*>(src);
  while (bytes) {
    const ssize_t r = ::pwrite(fd, p, bytes, off_t(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    p += r;
    bytes -= size_t(r);
    off += uint64_t(r);
  }
  return true;
}

// Open + validate like InputStream::open (stream.cpp:219-257).
int open_stream(const char* path, int expected_kind, Fd& f, Header& h, gwg_status* st) {
  f.fd = ::open(path, O_RDONLY);
  if (f.fd < 0)
    return set_status(st, GWG_IO, -1, -1, "cannot open %s: %s", path, std::strerror(errno));
  struct stat sb;
  if (::fstat(f.fd, &sb) != 0)
    return set_status(st, GWG_IO, -1, -1, "cannot stat %s", path);
  if (uint64_t(sb.st_size) < kHeader)
    return set_status(st, GWG_IO, -1, -1, "%s is shorter than the header (%lld of 64 bytes)",
                      path, (long long)sb.st_size);
  unsigned char b[kHeader];
  if (!pread_all(f.fd, b, kHeader, 0))
    return set_status(st, GWG_IO, -1, -1, "cannot read the header of %s", path);
  if (std::memcmp(b, "GWG1", 4) != 0)
    return set_status(st, GWG_IO, -1, -1, "bad magic in %s (not a GWG1 stream)", path);
  const int version = b[4] | (b[5] << 8);
  if (version != 1)
    return set_status(st, GWG_IO, -1, -1, "unsupported stream version %d in %s (expected 1)",
                      version, path);
  if (b[6] < 1 || b[6] > 4)
    return set_status(st, GWG_IO, -1, -1, "unknown stream kind %d in %s", b[6], path);
  if (b[7] != 0)
    return set_status(st, GWG_IO, -1, -1, "unsupported element type %d in %s", b[7], path);
  if (b[32] != 0)
    return set_status(st, GWG_IO, -1, -1, "unsupported layout %d in %s", b[32], path);
  h.kind = b[6];
  for (int d = 0; d < 3; ++d) {
    h.dims[d] = 0;
    for (int q = 0; q < 8; ++q) h.dims[d] |= uint64_t(b[8 + 8 * d + q]) << (8 * q);
  }
  h.complete = b[33] == 0;
  const uint64_t min_cols = h.kind == 4 ? 0 : 1;
  if (h.dims[0] < 1 || h.dims[1] < min_cols)
    return set_status(st, GWG_IO, -1, -1, "non-positive dims in %s", path);
  if (h.kind == 3 ? h.dims[2] < 1 : h.dims[2] != 0)
    return set_status(st, GWG_IO, -1, -1, "bad third dim in %s", path);
  if (expected_kind && h.kind != expected_kind)
    return set_status(st, GWG_IO, -1, -1, "%s holds a %s, expected a %s", path,
                      kind_name(h.kind), kind_name(expected_kind));
  if (!h.complete)
    return set_status(st, GWG_IO, -1, -1, "%s was never finalized by its writer", path);
  const uint64_t want = kHeader + payload_bytes(h);
  if (uint64_t(sb.st_size) != want)
    return set_status(st, GWG_IO, -1, -1, "%s has %lld bytes, header promises %llu", path,
                      (long long)sb.st_size, (unsigned long long)want);
  return GWG_OK;
}

}  // namespace

extern "C" {

int32_t gwg_stream_info(const char* path, int32_t* kind, int64_t* dims, int32_t* complete,
                        gwg_status* st) {
  clear_status(st);
  Fd f;
  f.fd = ::open(path, O_RDONLY);
  if (f.fd < 0)
    return set_status(st, GWG_IO, -1, -1, "cannot open %s: %s", path, std::strerror(errno));
  unsigned char b[kHeader];
  if (!pread_all(f.fd, b, kHeader, 0) || std::memcmp(b, "GWG1", 4) != 0)
    return set_status(st, GWG_IO, -1, -1, "bad magic in %s (not a GWG1 stream)", path);
  if (kind) *kind = b[6];
  for (int d = 0; d < 3 && dims; ++d) {
    uint64_t v = 0;
    for (int q = 0; q < 8; ++q) v |= uint64_t(b[8 + 8 * d + q]) << (8 * q);
    dims[d] = int64_t(v);
  }
  if (complete) *complete = b[33] == 0;
  return GWG_OK;
}

int32_t gwg_set_traits_file(gwg_engine* e, const char* traits_path, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  Fd f;
  Header h;
  if (int rc = open_stream(traits_path, 2, f, h, st)) return rc;
  if (int64_t(h.dims[0]) != e->n)
    return set_status(st, GWG_DIMENSION, -1, -1,
                      "trait stream rows (%llu) disagree with the kinship dimension (%lld)",
                      (unsigned long long)h.dims[0], (long long)e->n);
  const int64_t t = int64_t(h.dims[1]);
  std::vector<double> y(size_t(e->n) * t), h2(t), s2(t);
  if (!pread_all(f.fd, y.data(), y.size() * 8, kHeader) ||
      !pread_all(f.fd, h2.data(), t * 8, kHeader + y.size() * 8) ||
      !pread_all(f.fd, s2.data(), t * 8, kHeader + (y.size() + t) * 8))
    return set_status(st, GWG_IO, -1, -1, "short read in %s", traits_path);
  return gwg_set_traits(e, t, y.data(), h2.data(), s2.data(), GWG_HOST, 0, st);
}

}  // extern "C"


extern "C" {

int32_t gwg_run_grid_files(gwg_engine* e, const char* snps_path, int32_t snps_rotated,
                           const char* out_path, const gwg_run_options* opts,
                           gwg_counters* counters, gwg_status* st) {
  NvtxRange nvtx_("gwg_run_grid_files");
  clear_status(st);
  if (int rc = check_engine(e, st, false)) return rc;  // joined before the first rotation
  if (!e->have_traits)
    return set_status(st, GWG_DIMENSION, -1, -1, "traits must be installed first");
  Fd in;
  Header hin;
  if (int rc = open_stream(snps_path, 1, in, hin, st)) return rc;
  const int64_t n = e->n, t = e->t, p = e->p;
  if (int64_t(hin.dims[0]) != n)
    return set_status(st, GWG_DIMENSION, -1, -1,
                      "variant stream rows (%llu) disagree with the kinship dimension (%lld)",
                      (unsigned long long)hin.dims[0], (long long)n);
  const int64_t m = int64_t(hin.dims[1]);
  const int64_t mb = opts && opts->mb > 0 ? std::min(opts->mb, m) : default_slab(e, m);
  const auto wall0 = std::chrono::steady_clock::now();

  // Output: header marked incomplete, payload preallocated (stream.cpp:319-336).
  Fd out;
  out.fd = ::open(out_path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (out.fd < 0)
    return set_status(st, GWG_IO, -1, -1, "cannot create %s: %s", out_path,
                      std::strerror(errno));
  Header hout;
  hout.kind = 3;
  hout.dims[0] = uint64_t(m);
  hout.dims[1] = uint64_t(t);
  hout.dims[2] = uint64_t(p);
  hout.complete = false;
  unsigned char hb_[kHeader];
  encode(hout, hb_);
  if (!pwrite_all(out.fd, hb_, kHeader, 0) ||
      ::ftruncate(out.fd, off_t(kHeader + payload_bytes(hout))) != 0)
    return set_status(st, GWG_IO, -1, -1, "cannot size %s", out_path);

  const int fd_in = in.fd, fd_out = out.fd;
  PipeSpec sp;
  sp.m = m;
  sp.mb = mb;
  sp.rotated = snps_rotated != 0;
  sp.layout = GWG_LAYOUT_STREAM;
  sp.read_fn = [&](int64_t i0, int64_t rows, void* dst) {
    return pread_all(fd_in, dst, size_t(n) * rows * 8, kHeader + uint64_t(i0) * n * 8);
  };
  // write_result_cells (stream.cpp:414-438): t contiguous runs per slab
  sp.write_fn = [&](int64_t i0, int64_t rows, const double* src) {
    const size_t run = size_t(rows) * p * 8;
    for (int64_t j = 0; j < t; ++j)
      if (!pwrite_all(fd_out, src + size_t(j) * rows * p, run,
                      kHeader + (uint64_t(j) * m + i0) * p * 8))
        return false;
    return true;
  };
  e->i8_input = false;
  PipeStats ps;
  const int rc = run_pipeline(e, sp, &ps, st);
  const uint64_t loaded = ps.loaded, stored = ps.stored;
  e->counters.io_stall_ms += ps.stall_ms;
  if (rc != GWG_OK || ps.io_error) {  // the failed run's epoch ends here
    e->epoch_open = false;
    e->timings_used = e->timings_first = 0;
  }
  if (ps.io_error)
    return set_status(st, GWG_IO, -1, -1, ps.io_error == 1 ? "short read in %s" : "short write to %s",
                      ps.io_error == 1 ? snps_path : out_path);
  if (rc != GWG_OK) {
    e->epoch_open = false;
    return rc;
  }
  const int erc = end_epoch(e, st);
  e->counters.bytes_loaded += loaded;
  e->counters.bytes_stored += stored;
  e->counters.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  if (counters) *counters = e->counters;
  // A failing cell leaves the output incomplete, like the reference (the
  // exception skips out.finalize(), grid.cpp:640; test_grid.cpp:769-771).
  if (erc) return erc;
  const unsigned char zero = 0;
  if (!pwrite_all(fd_out, &zero, 1, 33))
    return set_status(st, GWG_IO, -1, -1, "cannot finalize %s", out_path);
  return GWG_OK;
}

}  // extern "C"
