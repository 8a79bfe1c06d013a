// pipeline.cu — run_grid's out-of-core slab traversal on the device
// (gwg_run_grid).
//
// Reference: run_grid (proj/src/grid.cpp:454-641) streams SNP slabs through
// pipeline_run (proj/include/gwgrid/pipeline.hpp:78-137): two workspaces, a
// prefetch agent loading slab s+2 and a writeback agent storing slab s while
// the caller computes slab s+1; stall = the compute side's waits (tail
// stores included).  Here:
//
//   H2D stream : raw slab s -> raw[s % 2] (pinned source: the caller's array
//                or a staging buffer a reader thread filled)
//   compute    : rotate (FP64 DMMA, or the exact int8 path for genotype
//                codes) -> grid -> optional checksum, into out[s % 2]
//   D2H stream : out[s % 2] -> the caller's pinned array, or one of `ring`
//                pinned result buffers that a writer thread hands to the
//                sink / file writer / pageable copy
//
// CUDA events hand each buffer from one agent to the next exactly as the
// reference's futures do; nothing is ever read while being written.  The
// stall is measured on the device: the compute stream's gaps between slabs
// (first load included) plus the host-side tail after the last compute.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "engine_internal.cuh"

using namespace gwg_host;

namespace {

// Binary hand-off of one host buffer between the coordinator and an agent.
struct Slot {
  std::mutex mu;
  std::condition_variable cv;
  int64_t ready = -1;  // slab whose data the consumer may take
  int64_t freed = -1;  // last slab the consumer released
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

cudaError_t ensure_events(std::vector<cudaEvent_t>& v, size_t count, unsigned flags) {
  while (v.size() < count) {
    cudaEvent_t ev;
    cudaError_t err = cudaEventCreateWithFlags(&ev, flags);
    if (err != cudaSuccess) return err;
    v.push_back(ev);
  }
  return cudaSuccess;
}

}  // namespace

namespace gwg_host {

int run_pipeline(gwg_engine* e, const PipeSpec& sp, PipeStats* stats, gwg_status* st) {
  const int64_t n = e->n, t = e->t, p = e->p, m = sp.m, mb = sp.mb;
  const bool i8 = sp.fmt == GWG_FORMAT_I8;
  const size_t elem = i8 ? 1 : sizeof(double);
  const bool staged_in = sp.x_direct == nullptr;
  const bool staged_out = sp.b_direct == nullptr;
  const int nb = sp.dbuf ? 2 : 1;                       // device buffers per side
  const int ring = staged_out ? std::max(2, std::min(sp.ring, 8)) : 0;
  const size_t slab_in = size_t(n) * mb * elem;
  const size_t slab_out = size_t(mb) * t * p * sizeof(double);
  const int64_t slabs = ceil_div(m, mb);
  const int64_t m_total = kKeyStride;                   // error keys: j * kKeyStride + i

  // ---- buffers (pinned staging cached by the engine) ----
  if (staged_in)
    for (int b = 0; b < 2; ++b) GWG_CUDA_TRY(e->pin_x[b].ensure(slab_in));
  if (int(e->pin_res.size()) < ring) e->pin_res.resize(ring);
  for (int b = 0; b < ring; ++b) GWG_CUDA_TRY(e->pin_res[b].ensure(slab_out));
  for (int b = 0; b < nb; ++b) {
    if (i8)
      GWG_CUDA_TRY(e->raw8[b].ensure(slab_in));
    else
      GWG_CUDA_TRY(e->raw[b].ensure(size_t(raw_ld(e)) * mb * sizeof(double)));
    GWG_CUDA_TRY(e->out[b].ensure(slab_out));
  }
  if (sp.rotated || !rotated_x_unused(e))
    GWG_CUDA_TRY(e->rot.ensure(size_t(e->np) * mb * sizeof(double)));
  GWG_CUDA_TRY(e->rot_sq.ensure(size_t(e->np) * mb * sizeof(double)));
  if (sp.checksum && !e->csum.ptr) {  // the accumulator starts at zero
    GWG_CUDA_TRY(e->csum.ensure(sizeof(unsigned long long)));
    GWG_CUDA_TRY(cudaMemsetAsync(e->csum.ptr, 0, sizeof(unsigned long long), e->comp));
  }
  // per slab: [start (after the waits), rotated, grid done, end (checksum done)]
  GWG_CUDA_TRY(ensure_events(e->slab_events, size_t(4 * slabs + 1), cudaEventDefault));
  // host hand-offs: [0,1] staging slab consumed by its H2D, [2, 2+ring) result
  // buffer filled by its D2H
  GWG_CUDA_TRY(ensure_events(e->pipe_events, size_t(2 + ring), cudaEventDisableTiming));
  cudaEvent_t* ev = e->slab_events.data();
  cudaEvent_t ev_begin = ev[4 * slabs];
  cudaEvent_t* ev_hx = e->pipe_events.data();
  cudaEvent_t* ev_res = e->pipe_events.data() + 2;

  if (int rc = begin_epoch(e, st)) return rc;
  for (int b = 0; b < 2; ++b) {  // fresh pipeline: every buffer starts free
    GWG_CUDA_TRY(cudaEventRecord(e->ev_rot_done[b], e->comp));
    GWG_CUDA_TRY(cudaEventRecord(e->ev_d2h_done[b], e->comp));
    GWG_CUDA_TRY(cudaEventRecord(e->ev_h2d[b], e->comp));
  }
  GWG_CUDA_TRY(cudaEventRecord(ev_begin, e->comp));
  cudaStream_t up = sp.dbuf ? e->h2d : e->comp;
  cudaStream_t down = sp.dbuf ? e->d2h : e->comp;

  Slot xs[2];
  std::vector<Slot> rs(std::max(ring, 1));
  std::atomic<bool> abort{false};
  std::atomic<int> io_error{0};
  std::atomic<uint64_t> loaded{0}, stored{0};
  auto wake_all = [&] {
    for (auto& q : xs) q.cv.notify_all();
    for (auto& q : rs) q.cv.notify_all();
  };

  std::thread reader, writer;
  if (staged_in)
    reader = std::thread([&] {
      for (int64_t s = 0; s < slabs && !abort.load(); ++s) {
        const int b = int(s & 1);
        if (!xs[b].wait([&] { return xs[b].freed >= s - 2; }, abort)) return;
        if (s >= 2) cudaEventSynchronize(ev_hx[b]);  // the H2D of slab s-2 left it
        const int64_t i0 = s * mb, rows = std::min(mb, m - i0);
        if (!sp.read_fn(i0, rows, e->pin_x[b].ptr)) {
          io_error = 1;
          abort = true;
          wake_all();
          return;
        }
        loaded += uint64_t(n) * rows * elem;
        xs[b].publish(s);
      }
    });
  if (staged_out)
    writer = std::thread([&] {
      for (int64_t s = 0; s < slabs && !abort.load(); ++s) {
        const int b = int(s % ring);
        if (!rs[b].wait([&] { return rs[b].ready >= s; }, abort)) return;
        cudaEventSynchronize(ev_res[b]);
        const int64_t i0 = s * mb, rows = std::min(mb, m - i0);
        if (!sp.write_fn(i0, rows, static_cast<const double*>(e->pin_res[b].ptr))) {
          io_error = 2;
          abort = true;
          wake_all();
          return;
        }
        stored += uint64_t(rows) * t * p * 8;
        rs[b].release(s);
      }
    });

  // the split grid's trait-side build runs on the side stream from here on,
  // under the first slab's upload and rotation
  int rc = mark_trait_fork(e, sp.rotated, st);
  for (int64_t s = 0; s < slabs && rc == GWG_OK; ++s) {
    const int bd = int(s % nb), hb = int(s & 1);
    const int64_t il0 = s * mb, rows = std::min(mb, m - il0);
    if (staged_in && !xs[hb].wait([&] { return xs[hb].ready >= s; }, abort)) break;
    auto enqueue = [&]() -> int {
      // H2D once the rotation of slab s - nb released raw[bd]
      GWG_CUDA_TRY(cudaStreamWaitEvent(up, e->ev_rot_done[bd], 0));
      const char* src = staged_in ? static_cast<const char*>(e->pin_x[hb].ptr)
                                  : static_cast<const char*>(sp.x_direct) + size_t(il0) * n * elem;
      if (i8) {
        GWG_CUDA_TRY(cudaMemcpyAsync(e->raw8[bd].ptr, src, size_t(n) * rows, cudaMemcpyHostToDevice,
                                     up));
      } else if (raw_ld(e) == n) {
        // contiguous on both sides: one flat copy (a pitched copy of 8n-byte
        // rows measured 41 vs 55 GB/s over PCIe, and its longer H2D window
        // slowed the concurrent result D2H: c1 e2e 67 -> see DESIGN)
        GWG_CUDA_TRY(cudaMemcpyAsync(e->raw[bd].ptr, src, size_t(n) * rows * 8,
                                     cudaMemcpyHostToDevice, up));
      } else {
        GWG_CUDA_TRY(cudaMemcpy2DAsync(e->raw[bd].ptr, raw_ld(e) * 8, src, n * 8, n * 8, rows,
                                       cudaMemcpyHostToDevice, up));
      }
      if (!staged_in) loaded += uint64_t(n) * rows * elem;
      GWG_CUDA_TRY(cudaEventRecord(e->ev_h2d[bd], up));
      if (staged_in) GWG_CUDA_TRY(cudaEventRecord(ev_hx[hb], up));
      // compute once the slab landed and out[bd] drained
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->comp, e->ev_h2d[bd], 0));
      GWG_CUDA_TRY(cudaStreamWaitEvent(e->comp, e->ev_d2h_done[bd], 0));
      GWG_CUDA_TRY(cudaEventRecord(ev[4 * s], e->comp));
      if (sp.rotated) {
        GWG_CUDA_TRY(cudaMemcpy2DAsync(e->rot.ptr, e->np * 8, e->raw[bd].ptr, raw_ld(e) * 8, n * 8,
                                       rows, cudaMemcpyDeviceToDevice, e->comp));
        if (int r = square_rotated(e, rows, st)) return r;
      } else if (i8) {
        if (int r = rotate_snps_i8(e, static_cast<const int8_t*>(e->raw8[bd].ptr), rows, st))
          return r;
      } else if (int r = rotate_snps(e, e->raw[bd].d(), raw_ld(e), rows, st)) {
        return r;
      }
      GWG_CUDA_TRY(cudaEventRecord(e->ev_rot_done[bd], e->comp));
      GWG_CUDA_TRY(cudaEventRecord(ev[4 * s + 1], e->comp));
      const int64_t si = sp.layout == GWG_LAYOUT_NUMPY ? t : 1;
      const int64_t sj = sp.layout == GWG_LAYOUT_NUMPY ? 1 : rows;
      if (int r = launch_slab(e, e->rot.d(), e->rot_sq.d(), rows, sp.i0 + il0, m_total,
                              e->out[bd].d(), si, sj, st))
        return r;
      GWG_CUDA_TRY(cudaEventRecord(ev[4 * s + 2], e->comp));
      if (sp.checksum)
        if (int r = launch_checksum(e, e->out[bd].d(), rows, sp.layout, sp.i0 + il0, st)) return r;
      GWG_CUDA_TRY(cudaEventRecord(ev[4 * s + 3], e->comp));
      GWG_CUDA_TRY(cudaEventRecord(e->ev_comp[bd], e->comp));
      return GWG_OK;
    };
    if ((rc = enqueue()) != GWG_OK) break;
    if (staged_in) xs[hb].release(s);
    // D2H of the slab's results
    const int hr = staged_out ? int(s % ring) : 0;
    if (staged_out && !rs[hr].wait([&] { return rs[hr].freed >= s - ring; }, abort)) break;
    auto d2h = [&]() -> int {
      GWG_CUDA_TRY(cudaStreamWaitEvent(down, e->ev_comp[bd], 0));
      const size_t run = size_t(rows) * p * 8;
      if (staged_out) {
        GWG_CUDA_TRY(cudaMemcpyAsync(e->pin_res[hr].ptr, e->out[bd].ptr, run * t,
                                     cudaMemcpyDeviceToHost, down));
      } else if (sp.layout == GWG_LAYOUT_NUMPY) {
        GWG_CUDA_TRY(cudaMemcpyAsync(sp.b_direct + size_t(il0) * t * p, e->out[bd].ptr, run * t,
                                     cudaMemcpyDeviceToHost, down));
      } else {
        GWG_CUDA_TRY(cudaMemcpy2DAsync(sp.b_direct + size_t(il0) * p, size_t(sp.ldb) * p * 8,
                                       e->out[bd].ptr, run, run, t, cudaMemcpyDeviceToHost, down));
      }
      if (!staged_out) stored += uint64_t(rows) * t * p * 8;
      GWG_CUDA_TRY(cudaEventRecord(e->ev_d2h_done[bd], down));
      if (staged_out) GWG_CUDA_TRY(cudaEventRecord(ev_res[hr], down));
      return GWG_OK;
    };
    if ((rc = d2h()) != GWG_OK) break;
    if (staged_out) rs[hr].publish(s);
  }
  // the tail: stores still landing after the last compute are compute-side
  // waits too (pipeline.hpp:129-132)
  std::chrono::steady_clock::time_point tail0;
  bool tail_started = false;
  if (rc == GWG_OK && !abort.load()) {
    cudaEventSynchronize(ev[4 * (slabs - 1) + 3]);
    tail0 = std::chrono::steady_clock::now();
    tail_started = true;
  }
  if (rc != GWG_OK) abort = true;
  wake_all();
  if (reader.joinable()) reader.join();
  if (writer.joinable()) writer.join();
  cudaStreamSynchronize(e->h2d);
  cudaStreamSynchronize(e->comp);
  cudaStreamSynchronize(e->d2h);
  if (stats) {
    stats->loaded = loaded.load();
    stats->stored = stored.load();
    stats->io_error = io_error.load();
  }
  if (rc != GWG_OK) return rc;
  if (io_error.load()) return GWG_IO;
  GWG_CUDA_TRY(cudaGetLastError());
  double stall = 0.0;
  for (int64_t s = 0; s < slabs; ++s) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, s ? ev[4 * (s - 1) + 3] : ev_begin, ev[4 * s]) == cudaSuccess)
      stall += ms;
    if (cudaEventElapsedTime(&ms, ev[4 * s], ev[4 * s + 1]) == cudaSuccess)
      e->counters.rotate_ms += ms;
    if (cudaEventElapsedTime(&ms, ev[4 * s + 1], ev[4 * s + 2]) == cudaSuccess)
      e->counters.grid_kernel_ms += ms;
  }
  if (tail_started)
    stall += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tail0)
                 .count();
  if (stats) stats->stall_ms = stall;
  return GWG_OK;
}

int run_grid_impl(gwg_engine* e, int64_t m, const void* x_r_host, double* b_host,
                  const gwg_run_options* opts, gwg_counters* counters, gwg_status* st) {
  if (!e->have_traits)
    return set_status(st, GWG_DIMENSION, -1, -1, "gwg_set_traits must come first");
  const bool sink = opts && opts->sink;
  if (m < 1 || !x_r_host || (!b_host && !sink))
    return set_status(st, GWG_DIMENSION, -1, -1, "bad run_grid arguments (m=%lld)",
                      (long long)m);
  const int layout = opts ? opts->layout : GWG_LAYOUT_NUMPY;
  if (layout != GWG_LAYOUT_NUMPY && layout != GWG_LAYOUT_STREAM)
    return set_status(st, GWG_DIMENSION, -1, -1, "unknown layout %d", layout);
  const int fmt = opts ? opts->snp_format : GWG_FORMAT_F64;
  if (fmt != GWG_FORMAT_F64 && fmt != GWG_FORMAT_I8)
    return set_status(st, GWG_DIMENSION, -1, -1, "unknown SNP format %d", fmt);
  const int64_t i0 = opts ? opts->i0 : 0;
  if (i0 < 0) return set_status(st, GWG_DIMENSION, -1, -1, "negative i0 (%lld)", (long long)i0);
  const int64_t ldb = opts && opts->ldb > 0 ? opts->ldb : m;
  if (ldb < m)
    return set_status(st, GWG_DIMENSION, -1, -1, "ldb (%lld) < m (%lld)", (long long)ldb,
                      (long long)m);
  if (fmt == GWG_FORMAT_I8 && e->snp_coding == GWG_SNP_GENOTYPES && e->n >= kMaxGenotypeN)
    return set_status(st, GWG_DIMENSION, -1, -1,
                      "genotype coding needs n < 132,000 (exact int32 accumulation)");
  const auto wall0 = std::chrono::steady_clock::now();
  const int64_t n = e->n, t = e->t, p = e->p;
  const size_t elem = fmt == GWG_FORMAT_I8 ? 1 : 8;
  e->i8_input = fmt == GWG_FORMAT_I8;

  PipeSpec sp;
  sp.m = m;
  sp.i0 = i0;
  sp.mb = opts && opts->mb > 0 ? std::min(opts->mb, m) : default_slab(e, m);
  sp.fmt = fmt;
  sp.layout = layout;
  sp.dbuf = opts ? opts->double_buffer != 0 : true;
  sp.ring = opts && opts->ring > 0 ? opts->ring : 2;
  sp.checksum = opts && opts->checksum;
  sp.ldb = ldb;
  // Page-locked caller buffers stream directly; anything else goes through
  // the engine's own pinned staging on reader/writer threads (registering
  // arbitrary user memory in place is unsafe when a neighbouring allocation
  // already registered part of its pages).
  const size_t x_bytes = size_t(n) * m * elem;
  const char* xc = static_cast<const char*>(x_r_host);
  if (is_pinned_host(xc) && is_pinned_host(xc + x_bytes - 1)) {
    sp.x_direct = x_r_host;
  } else {
    sp.read_fn = [=](int64_t il0, int64_t rows, void* dst) {
      parallel_copy(dst, xc + size_t(il0) * n * elem, size_t(n) * rows * elem);
      return true;
    };
  }
  if (sink) {
    const gwg_result_sink fn = opts->sink;
    void* user = opts->sink_user;
    sp.write_fn = [=](int64_t il0, int64_t rows, const double* cells) {
      return fn(user, i0 + il0, rows, cells) == 0;
    };
  } else {
    const size_t b_bytes =
        (layout == GWG_LAYOUT_NUMPY ? size_t(m) * t : size_t(ldb) * (t - 1) + m) * p * 8;
    const char* bc = reinterpret_cast<const char*>(b_host);
    if (is_pinned_host(bc) && is_pinned_host(bc + b_bytes - 1)) {
      sp.b_direct = b_host;
    } else {
      sp.write_fn = [=](int64_t il0, int64_t rows, const double* src) {
        if (layout == GWG_LAYOUT_NUMPY) {
          parallel_copy(b_host + size_t(il0) * t * p, src, size_t(rows) * t * p * 8);
        } else {
          for (int64_t j = 0; j < t; ++j)
            std::memcpy(b_host + (size_t(j) * ldb + il0) * p, src + size_t(j) * rows * p,
                        size_t(rows) * p * 8);
        }
        return true;
      };
    }
  }
  PipeStats ps;
  const int rc = run_pipeline(e, sp, &ps, st);
  e->counters.bytes_loaded += ps.loaded;
  e->counters.bytes_stored += ps.stored;
  e->counters.io_stall_ms += ps.stall_ms;
  if (rc != GWG_OK || ps.io_error) {  // the failed run's epoch ends here
    e->epoch_open = false;
    e->timings_used = e->timings_first = 0;
  }
  if (ps.io_error == 2 && sink)
    return set_status(st, GWG_IO, -1, -1, "result sink aborted the run");
  if (rc != GWG_OK) {
    e->epoch_open = false;
    return rc;
  }
  const int erc = end_epoch(e, st);  // trait, genotype and cell errors
  if (sp.checksum) {
    unsigned long long sum = 0;
    GWG_CUDA_TRY(cudaMemcpy(&sum, e->csum.ptr, sizeof(sum), cudaMemcpyDeviceToHost));
    e->counters.checksum = sum;
    e->counters.checksum_cells = e->csum_cells;
  }
  e->counters.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  if (counters) *counters = e->counters;
  return erc;
}

}  // namespace gwg_host

extern "C" {

int32_t gwg_run_grid(gwg_engine* e, int64_t m, const void* x_r_host, double* b_host,
                     const gwg_run_options* opts, gwg_counters* counters, gwg_status* st) {
  NvtxRange nvtx_("gwg_run_grid");
  clear_status(st);
  // no join here: the pipeline joins trait work still on the side stream right
  // before the first slab's rotation, so the first uploads overlap it
  if (int rc = check_engine(e, st, false)) return rc;
  return run_grid_impl(e, m, x_r_host, b_host, opts, counters, st);
}

int32_t gwg_wait_stream(gwg_engine* e, void* stream, gwg_status* st) {
  clear_status(st);
  // no join: the trait side forks from the compute stream after this wait
  if (int rc = check_engine(e, st, false)) return rc;
  if (!e->ev_wait) GWG_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_wait, cudaEventDisableTiming));
  GWG_CUDA_TRY(cudaEventRecord(e->ev_wait, static_cast<cudaStream_t>(stream)));
  GWG_CUDA_TRY(cudaStreamWaitEvent(e->comp, e->ev_wait, 0));
  return GWG_OK;
}

int32_t gwg_signal_stream(gwg_engine* e, void* stream, gwg_status* st) {
  clear_status(st);
  if (int rc = check_engine(e, st)) return rc;
  if (!e->ev_signal)
    GWG_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_signal, cudaEventDisableTiming));
  GWG_CUDA_TRY(cudaEventRecord(e->ev_signal, e->comp));
  GWG_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e->ev_signal, 0));
  return GWG_OK;
}

}  // extern "C"
