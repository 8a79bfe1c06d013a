// group.cu — one process driving several GPUs (gwg_group_* in
// include/gwgrid_cuda.h).
//
// The reference parallelises run_grid over CPU workers (CT: a shared block
// FIFO, IT: static slab ownership k = w mod workers, proj/src/grid.cpp:519-639)
// in one address space.  The device analogue shards the SNP axis m into
// contiguous column ranges, one per GPU:
//   * shared operands reach the first device from the host once, and every
//     other device copies them device-to-device (peer copies over NVLink /
//     NVSwitch, cudaMemcpyPeer through UVA): Z and lambda, the ROTATED
//     covariates X_L' and traits Y' (so the O(n^2) rotations run once), h2
//     and sigma2; each device then builds its own trait contexts;
//   * each device streams its own shard through its own pinned buffers and
//     PCIe link from its own host thread (the IT discipline at device
//     granularity), writing disjoint result rows;
//   * no other collective: cells are independent, results land at global
//     positions, error coordinates are global.  Because every kernel's
//     reduction order is fixed per cell, the grid is bitwise the same for any
//     device count (tested), and so is the order-independent checksum.
#include <algorithm>
#include <thread>
#include <vector>

#include "engine_internal.cuh"

using namespace gwg_host;

struct gwg_group {
  std::vector<gwg_engine*> engines;
  std::vector<int> devices;
  cudaEvent_t ready = nullptr;  // on the first device: its shared operands are in place
};

namespace {

int group_ok(gwg_group* g, gwg_status* st) {
  if (!g || g->engines.empty()) return set_status(st, GWG_DIMENSION, -1, -1, "null device group");
  return GWG_OK;
}

// After engine 0 queued an install: every other engine's stream waits for it
// (cross-device event wait, no host round trip) before its peer copies.
int publish_from_first(gwg_group* g, gwg_status* st) {
  gwg_engine* e0 = g->engines[0];
  GWG_CUDA_TRY(cudaSetDevice(e0->device));
  GWG_CUDA_TRY(join_side(e0));  // e0's trait work may still be on its side stream
  GWG_CUDA_TRY(cudaEventRecord(g->ready, e0->comp));
  for (size_t k = 1; k < g->engines.size(); ++k) {
    GWG_CUDA_TRY(cudaSetDevice(g->engines[k]->device));
    GWG_CUDA_TRY(cudaStreamWaitEvent(g->engines[k]->comp, g->ready, 0));
  }
  return GWG_OK;
}

}  // namespace

extern "C" {

gwg_group* gwg_group_create(const int32_t* devices, int32_t count, int64_t n, int64_t p,
                            gwg_status* st) {
  clear_status(st);
  if (!devices || count < 1) {
    set_status(st, GWG_DIMENSION, -1, -1, "a device group needs at least one device");
    return nullptr;
  }
  auto* g = new gwg_group();
  for (int32_t k = 0; k < count; ++k) {
    gwg_engine* e = gwg_engine_create(devices[k], n, p, st);
    if (!e) {
      gwg_group_destroy(g);
      return nullptr;
    }
    g->engines.push_back(e);
    g->devices.push_back(devices[k]);
  }
  // direct peer access where the fabric allows it (NVLink on HGX); copies
  // fall back to staging through the host otherwise
  for (int a : g->devices)
    for (int b : g->devices) {
      int can = 0;
      if (a != b && cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
        cudaSetDevice(a);
        if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already on
      }
    }
  cudaSetDevice(g->devices[0]);
  if (cudaEventCreateWithFlags(&g->ready, cudaEventDisableTiming) != cudaSuccess) {
    set_status(st, GWG_CUDA, -1, -1, "cudaEventCreate failed");
    gwg_group_destroy(g);
    return nullptr;
  }
  return g;
}

void gwg_group_destroy(gwg_group* g) {
  if (!g) return;
  for (gwg_engine* e : g->engines) gwg_engine_destroy(e);
  if (g->ready) {
    cudaSetDevice(g->devices[0]);
    cudaEventDestroy(g->ready);
  }
  delete g;
}

int32_t gwg_group_size(const gwg_group* g) { return g ? int32_t(g->engines.size()) : 0; }

gwg_engine* gwg_group_engine(gwg_group* g, int32_t k) {
  if (!g || k < 0 || k >= int32_t(g->engines.size())) return nullptr;
  return g->engines[k];
}

int32_t gwg_group_set_spectrum(gwg_group* g, const double* basis, const double* lambda,
                               int32_t where, gwg_status* st) {
  clear_status(st);
  if (int rc = group_ok(g, st)) return rc;
  if (int rc = gwg_set_spectrum(g->engines[0], basis, lambda, where, st)) return rc;
  if (int rc = publish_from_first(g, st)) return rc;
  gwg_engine* e0 = g->engines[0];
  for (size_t k = 1; k < g->engines.size(); ++k) {  // broadcast: peer copies
    gwg_engine* e = g->engines[k];
    GWG_CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = set_spectrum_impl(e, e0->basis.d(), e0->np, e0->lambda.d(), GWG_DEVICE, st))
      return rc;
  }
  return GWG_OK;
}

int32_t gwg_group_set_covariates(gwg_group* g, const double* xl, int32_t where, gwg_status* st) {
  clear_status(st);
  if (int rc = group_ok(g, st)) return rc;
  if (int rc = gwg_set_covariates(g->engines[0], xl, where, st)) return rc;
  if (int rc = publish_from_first(g, st)) return rc;
  gwg_engine* e0 = g->engines[0];
  for (size_t k = 1; k < g->engines.size(); ++k) {  // X_L' already rotated on device 0
    gwg_engine* e = g->engines[k];
    GWG_CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = set_covariates_impl(e, e0->xl_rot.d(), e0->np, GWG_DEVICE, true, st)) return rc;
  }
  return GWG_OK;
}

int32_t gwg_group_set_traits(gwg_group* g, int64_t t, const double* y, const double* h2,
                             const double* sigma2, int32_t where, int32_t is_rotated,
                             gwg_status* st) {
  clear_status(st);
  if (int rc = group_ok(g, st)) return rc;
  gwg_engine* e0 = g->engines[0];
  if (int rc = gwg_set_traits(e0, t, y, h2, sigma2, where, is_rotated, st)) return rc;
  if (int rc = publish_from_first(g, st)) return rc;
  for (size_t k = 1; k < g->engines.size(); ++k) {
    // Y' rotated once on device 0 and broadcast; h2 / sigma2 from wherever
    // the caller keeps them (host copies spare the others a range round trip)
    gwg_engine* e = g->engines[k];
    GWG_CUDA_TRY(cudaSetDevice(e->device));
    const bool host_scalars = where == GWG_HOST;
    if (int rc = set_traits_impl(e, t, e0->y_rot.d(), e0->np, GWG_DEVICE,
                                 host_scalars ? h2 : e0->h2.d(),
                                 host_scalars ? sigma2 : e0->sigma2.d(),
                                 host_scalars ? GWG_HOST : GWG_DEVICE, true, st))
      return rc;
  }
  return GWG_OK;
}

int32_t gwg_group_set_snp_coding(gwg_group* g, int32_t coding, gwg_status* st) {
  clear_status(st);
  if (int rc = group_ok(g, st)) return rc;
  for (gwg_engine* e : g->engines)
    if (int rc = gwg_set_snp_coding(e, coding, st)) return rc;
  return GWG_OK;
}

int32_t gwg_group_set_option(gwg_group* g, int32_t option, int64_t value, gwg_status* st) {
  clear_status(st);
  if (int rc = group_ok(g, st)) return rc;
  for (gwg_engine* e : g->engines)
    if (int rc = gwg_set_option(e, option, value, st)) return rc;
  return GWG_OK;
}

int32_t gwg_group_shards(const gwg_group* g, int64_t m, int64_t* bounds) {
  if (!g || !bounds || m < 0) return GWG_DIMENSION;
  const int64_t count = int64_t(g->engines.size());
  for (int64_t k = 0; k <= count; ++k) bounds[k] = k * m / count;  // balanced, contiguous
  return GWG_OK;
}

int32_t gwg_group_run_grid(gwg_group* g, int64_t m, const void* x_r_host, double* b_host,
                           const gwg_run_options* opts, gwg_counters* counters,
                           gwg_status* st) {
  NvtxRange nvtx_("gwg_group_run_grid");
  clear_status(st);
  if (int rc = group_ok(g, st)) return rc;
  const bool sink = opts && opts->sink;
  if (m < 1 || !x_r_host || (!b_host && !sink))
    return set_status(st, GWG_DIMENSION, -1, -1, "bad run_grid arguments (m=%lld)",
                      (long long)m);
  const size_t count = g->engines.size();
  for (gwg_engine* e : g->engines)
    if (!e->have_traits)
      return set_status(st, GWG_DIMENSION, -1, -1, "gwg_group_set_traits must come first");
  std::vector<int64_t> bounds(count + 1);
  gwg_group_shards(g, m, bounds.data());
  gwg_run_options base{};
  base.layout = GWG_LAYOUT_NUMPY;
  base.double_buffer = 1;
  if (opts) base = *opts;
  const int64_t t = g->engines[0]->t, p = g->engines[0]->p, n = g->engines[0]->n;
  const size_t elem = base.snp_format == GWG_FORMAT_I8 ? 1 : 8;
  const int64_t ldb = base.ldb > 0 ? base.ldb : m;
  std::vector<gwg_counters> cnt(count);
  std::vector<gwg_status> sts(count);
  std::vector<int> rcs(count, GWG_OK);
  std::vector<std::thread> th;
  for (size_t k = 0; k < count; ++k) {
    const int64_t a = bounds[k], mk = bounds[k + 1] - bounds[k];
    if (mk == 0) continue;
    th.emplace_back([&, k, a, mk] {
      gwg_engine* e = g->engines[k];
      clear_status(&sts[k]);
      cudaSetDevice(e->device);
      gwg_run_options o = base;
      o.i0 = base.i0 + a;
      o.ldb = ldb;
      const void* x = static_cast<const char*>(x_r_host) + size_t(a) * n * elem;
      double* b = b_host ? b_host + (o.layout == GWG_LAYOUT_NUMPY ? size_t(a) * t * p
                                                                   : size_t(a) * p)
                         : nullptr;
      rcs[k] = run_grid_impl(e, mk, x, b, &o, &cnt[k], &sts[k]);
    });
  }
  for (auto& x : th) x.join();
  // counters: additive buckets summed, wall time and stall the slowest device's
  gwg_counters tot{};
  for (size_t k = 0; k < count; ++k) {
    const gwg_counters& c = cnt[k];
    tot.preloop_flops += c.preloop_flops;
    tot.loop_flops += c.loop_flops;
    tot.grid_flops += c.grid_flops;
    tot.bytes_loaded += c.bytes_loaded;
    tot.bytes_stored += c.bytes_stored;
    tot.context_builds += c.context_builds;
    tot.kernel_launches += c.kernel_launches;
    tot.grid_kernel_ms += c.grid_kernel_ms;
    tot.rotate_ms += c.rotate_ms;
    tot.wall_ms = std::max(tot.wall_ms, c.wall_ms);
    tot.linear_ms += c.linear_ms;
    tot.quad_ms += c.quad_ms;
    tot.sbr_flops += c.sbr_flops;
    tot.sbr_terms = std::max(tot.sbr_terms, c.sbr_terms);
    tot.io_stall_ms = std::max(tot.io_stall_ms, c.io_stall_ms);
    tot.checksum += c.checksum;  // wrapping: the sum over all cells
    tot.checksum_cells += c.checksum_cells;
  }
  if (counters) *counters = tot;
  // errors: a trait failure (-1, j) first (lowest j), then the first failing
  // cell of the whole grid in trait-major order, then anything else by device
  int best = -1;
  auto rank_of = [&](size_t k) -> int {
    if (rcs[k] != GWG_NOT_POSITIVE_DEFINITE) return 2;
    return sts[k].snp_index < 0 ? 0 : 1;
  };
  for (size_t k = 0; k < count; ++k) {
    if (rcs[k] == GWG_OK) continue;
    if (best < 0) {
      best = int(k);
      continue;
    }
    const int rk = rank_of(k), rb = rank_of(size_t(best));
    const gwg_status &a = sts[k], &b = sts[best];
    if (rk < rb || (rk == rb && rk < 2 &&
                    (a.trait_index < b.trait_index ||
                     (a.trait_index == b.trait_index && a.snp_index < b.snp_index))))
      best = int(k);
  }
  if (best >= 0) {
    if (st) *st = sts[best];
    return rcs[best];
  }
  return GWG_OK;
}

}  // extern "C"
