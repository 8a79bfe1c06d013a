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

bool pread_all(int fd, void* dst, size_t bytes, uint64_t off) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, bytes, off_t(off));
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

// A binary semaphore per buffer, for the reader/writer hand-offs.
struct Slot {
  std::mutex mu;
  std::condition_variable cv;
  int64_t ready = -1;  // slab index whose data is ready for the consumer
  int64_t freed = -1;  // last slab index the consumer released
  void publish(int64_t s) {
    { std::lock_guard<std::mutex> l(mu); ready = s; }
    cv.notify_all();
  }
  void release(int64_t s) {
    { std::lock_guard<std::mutex> l(mu); freed = s; }
    cv.notify_all();
  }
  template <class Pred>
  bool wait(Pred pred, const std::atomic<bool>& abort) {
    std::unique_lock<std::mutex> l(mu);
    cv.wait(l, [&] { return pred() || abort.load(); });
    return !abort.load();
  }
};

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

namespace gwg_host {

// The staged slab pipeline shared by the file legs and by gwg_run_grid on
// pageable host memory: a reader thread fills pinned hx[s%2] (read_fn), the
// coordinator runs H2D -> rotate (or square, for rotated input) -> fused grid
// -> D2H into pinned hres[s%2], a writer thread drains it (write_fn).  CUDA
// events hand buffer ownership between the three agents, exactly the
// two-workspace discipline of pipeline_run (pipeline.hpp:62-137).
int staged_pipeline(gwg_engine* e, int64_t m, int64_t mb, bool rotated, int out_layout,
                    const SlabRead& read_fn, const SlabWrite& write_fn, uint64_t* loaded_out,
                    uint64_t* stored_out, int* io_error_out, gwg_status* st) {
  const int64_t n = e->n, t = e->t, p = e->p;
  double* hx[2] = {nullptr, nullptr};
  double* hres[2] = {nullptr, nullptr};
  struct Pinned {
    double** a;
    double** b;
    ~Pinned() {
      for (int i = 0; i < 2; ++i) {
        if (a[i]) cudaFreeHost(a[i]);
        if (b[i]) cudaFreeHost(b[i]);
      }
    }
  } pinned{hx, hres};
  for (int b = 0; b < 2; ++b) {
    GWG_CUDA_TRY(cudaMallocHost(&hx[b], size_t(n) * mb * sizeof(double)));
    GWG_CUDA_TRY(cudaMallocHost(&hres[b], size_t(mb) * t * p * sizeof(double)));
    GWG_CUDA_TRY(e->raw[b].ensure(size_t(raw_ld(e)) * mb * sizeof(double)));
    GWG_CUDA_TRY(e->out[b].ensure(size_t(mb) * t * p * sizeof(double)));
  }
  if (rotated || !rotated_x_unused(e))
    GWG_CUDA_TRY(e->rot.ensure(size_t(e->np) * mb * sizeof(double)));
  GWG_CUDA_TRY(e->rot_sq.ensure(size_t(e->np) * mb * sizeof(double)));
  if (int rc = reset_errors(e, st)) return rc;
  for (int b = 0; b < 2; ++b) {
    GWG_CUDA_TRY(cudaEventRecord(e->ev_rot_done[b], e->comp));
    GWG_CUDA_TRY(cudaEventRecord(e->ev_d2h_done[b], e->comp));
    GWG_CUDA_TRY(cudaEventRecord(e->ev_h2d[b], e->comp));
  }
  const int64_t slabs = ceil_div(m, mb);
  while (int64_t(e->slab_events.size()) < 2 * slabs) {
    cudaEvent_t ev;
    GWG_CUDA_TRY(cudaEventCreate(&ev));
    e->slab_events.push_back(ev);
  }
  Slot xs[2], rs[2];
  std::atomic<bool> abort{false};
  std::atomic<int> io_error{0};  // 1 = read, 2 = write
  std::atomic<uint64_t> loaded{0}, stored{0};
  auto wake_all = [&] {
    for (auto& q : xs) q.cv.notify_all();
    for (auto& q : rs) q.cv.notify_all();
  };

  std::thread reader([&] {
    for (int64_t s = 0; s < slabs && !abort.load(); ++s) {
      const int b = int(s & 1);
      // the H2D of slab s-2 out of hx[b] must have completed
      if (!xs[b].wait([&] { return xs[b].freed >= s - 2; }, abort)) return;
      if (s >= 2) cudaEventSynchronize(e->ev_h2d[b]);
      const int64_t i0 = s * mb, rows = std::min(mb, m - i0);
      if (!read_fn(i0, rows, hx[b])) {
        io_error = 1;
        abort = true;
        wake_all();
        return;
      }
      loaded += uint64_t(n) * rows * 8;
      xs[b].publish(s);
    }
  });
  std::thread writer([&] {
    for (int64_t s = 0; s < slabs && !abort.load(); ++s) {
      const int b = int(s & 1);
      if (!rs[b].wait([&] { return rs[b].ready >= s; }, abort)) return;
      cudaEventSynchronize(e->ev_d2h_done[b]);
      const int64_t i0 = s * mb, rows = std::min(mb, m - i0);
      if (!write_fn(i0, rows, hres[b])) {
        io_error = 2;
        abort = true;
        wake_all();
        return;
      }
      stored += uint64_t(rows) * t * p * 8;
      rs[b].release(s);
    }
  });

  int rc = GWG_OK;
  for (int64_t s = 0; s < slabs && rc == GWG_OK; ++s) {
    const int b = int(s & 1);
    const int64_t i0 = s * mb, rows = std::min(mb, m - i0);
    if (!xs[b].wait([&] { return xs[b].ready >= s; }, abort)) break;
    auto enqueue = [&]() -> int {
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->h2d, e->ev_rot_done[b], 0));
      GWG_CUDA_TRY(cudaMemcpy2DAsync(e->raw[b].ptr, raw_ld(e) * 8, hx[b], n * 8, n * 8, rows,
                                     cudaMemcpyHostToDevice, e->h2d));
      GWG_CUDA_TRY(cudaEventRecord(e->ev_h2d[b], e->h2d));
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->comp, e->ev_h2d[b], 0));
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->comp, e->ev_d2h_done[b], 0));
      if (rotated) {
        GWG_CUDA_TRY(cudaMemcpy2DAsync(e->rot.ptr, e->np * 8, e->raw[b].ptr, raw_ld(e) * 8,
                                       n * 8, rows, cudaMemcpyDeviceToDevice, e->comp));
        if (int r = square_rotated(e, rows, st)) return r;
      } else if (int r = rotate_snps(e, e->raw[b].d(), raw_ld(e), rows, st)) {
        return r;
      }
      GWG_CUDA_TRY(cudaEventRecord(e->ev_rot_done[b], e->comp));
      GWG_CUDA_TRY(cudaEventRecord(e->slab_events[2 * s], e->comp));
      const int64_t si = out_layout == GWG_LAYOUT_NUMPY ? t : 1;
      const int64_t sj = out_layout == GWG_LAYOUT_NUMPY ? 1 : rows;
      if (int r = launch_slab(e, e->rot.d(), e->rot_sq.d(), rows, i0, m, e->out[b].d(), si, sj,
                              st))
        return r;
      GWG_CUDA_TRY(cudaEventRecord(e->slab_events[2 * s + 1], e->comp));
      GWG_CUDA_TRY(cudaEventRecord(e->ev_comp[b], e->comp));
      return GWG_OK;
    };
    if ((rc = enqueue()) != GWG_OK) break;
    xs[b].release(s);
    // D2H into hres[b] once the writer released slab s-2
    if (!rs[b].wait([&] { return rs[b].freed >= s - 2; }, abort)) break;
    auto d2h = [&]() -> int {
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->d2h, e->ev_comp[b], 0));
      GWG_CUDA_TRY(cudaMemcpyAsync(hres[b], e->out[b].ptr, size_t(rows) * t * p * 8,
                                   cudaMemcpyDeviceToHost, e->d2h));
      GWG_CUDA_TRY(cudaEventRecord(e->ev_d2h_done[b], e->d2h));
      return GWG_OK;
    };
    if ((rc = d2h()) != GWG_OK) break;
    rs[b].publish(s);
  }
  if (rc != GWG_OK) abort = true;
  wake_all();
  reader.join();
  writer.join();
  cudaStreamSynchronize(e->h2d);
  cudaStreamSynchronize(e->comp);
  cudaStreamSynchronize(e->d2h);
  if (rc != GWG_OK) return rc;
  if (io_error_out) *io_error_out = io_error.load();
  if (io_error) return GWG_IO;
  GWG_CUDA_TRY(cudaGetLastError());
  for (int64_t s = 0; s < slabs; ++s) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e->slab_events[2 * s], e->slab_events[2 * s + 1]) ==
        cudaSuccess)
      e->counters.grid_kernel_ms += ms;
  }
  if (loaded_out) *loaded_out = loaded.load();
  if (stored_out) *stored_out = stored.load();
  return read_errors(e, st, false);
}

}  // namespace gwg_host

extern "C" {

int32_t gwg_run_grid_files(gwg_engine* e, const char* snps_path, int32_t snps_rotated,
                           const char* out_path, const gwg_run_options* opts,
                           gwg_counters* counters, gwg_status* st) {
  NvtxRange nvtx_("gwg_run_grid_files");
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
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
  SlabRead rd = [&](int64_t i0, int64_t rows, double* dst) {
    return pread_all(fd_in, dst, size_t(n) * rows * 8, kHeader + uint64_t(i0) * n * 8);
  };
  // write_result_cells (stream.cpp:414-438): t contiguous runs per slab
  SlabWrite wr = [&](int64_t i0, int64_t rows, const double* src) {
    const size_t run = size_t(rows) * p * 8;
    for (int64_t j = 0; j < t; ++j)
      if (!pwrite_all(fd_out, src + size_t(j) * rows * p, run,
                      kHeader + (uint64_t(j) * m + i0) * p * 8))
        return false;
    return true;
  };
  uint64_t loaded = 0, stored = 0;
  int io_error = 0;
  const int rc = staged_pipeline(e, m, mb, snps_rotated != 0, GWG_LAYOUT_STREAM, rd, wr,
                                 &loaded, &stored, &io_error, st);
  if (io_error)
    return set_status(st, GWG_IO, -1, -1, io_error == 1 ? "short read in %s" : "short write to %s",
                      io_error == 1 ? snps_path : out_path);
  if (rc != GWG_OK) return rc;
  e->counters.bytes_loaded += loaded;
  e->counters.bytes_stored += stored;
  e->counters.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  if (counters) *counters = e->counters;
  // A failing cell leaves the output incomplete, like the reference (the
  // exception skips out.finalize(), grid.cpp:640; test_grid.cpp:769-771).
  if (int r = raise_cell_error(e, m, st)) return r;
  const unsigned char zero = 0;
  if (!pwrite_all(fd_out, &zero, 1, 33))
    return set_status(st, GWG_IO, -1, -1, "cannot finalize %s", out_path);
  return GWG_OK;
}

}  // extern "C"
