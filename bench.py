"""Benchmark: GLS problems solved/sec on BASELINE.json configs[1] (c1).

c1: n=1000, p=4, m=100,000 SNPs per GPU, t=1,000 traits, FP64, synthetic
inputs from BASELINE.json's generators (one seed).  A step is one pass of the
hot path over one batch: rotate Y' = Z^T Y and X_R' = Z^T X_R on the device,
build every trait context, and solve all m x t cells (the eigendecomposition
is the one-off CPU preloop, outside the step, as in the paper).

  value  : inputs already resident in HBM (device pointers through the C ABI)
  e2e    : the same step through gwg_set_traits + gwg_run_grid with pinned HOST
           buffers (X_R as BASELINE's doubles): H2D of X_R and Y and D2H of
           every b_ij inside the timed region; e2e_int8 the same with the
           genotype codes as 1-byte int8 (GWG_FORMAT_I8)
  parity : the timed grid against the CPU oracle's full c1 grid (every cell)
  --impl reference : the reference's CPU path (oracle/: the restatement of
           gwgrid's compute_tile CT scheduler + OpenBLAS rotation) on the host
           cores over the same full c1 grid per step; it loads no engine code
           (inputs from the oracle library's copy of the generator).

Multi-GPU (torchrun): paper_1210_7683_b200.multi shards the SNP axis (weak
scaling: m SNPs per rank); Z, lambda, X_L, Y, h2 are broadcast once from rank
0 over NCCL; no data-path collective; timing is max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GLS problems solved/sec (m·t/s) at n=1000,p=4; FP64 TFLOP/s vs B200 peak"
PEAK_FP64_TFLOPS = 37.15  # measured DMMA.8x8x4 loop, profiles/r01_fp64_peak.txt
I8_SLICES = 7  # int8 slices of W per linear term (i8_core.cuh, slice_basis_kernel)
# int8 dense tensor peak measured on this pool's B200 (tools/i8_peak.cu:
# tcgen05.mma kind::i8 M128 N256 K32 from resident smem, warp-collective
# elected issue, 148 CTAs, 1965 MHz — the best of its issue modes; round 1's
# single-thread issue loop reached 4346); MEASURED_PEAKS.json has no int8 entry
PEAK_INT8_TOPS = 4462.0
PEAK_INT8_SOURCE = ("measured: tcgen05.mma.kind::i8 M128 N256 K32 issue loop (warp-elected) "
                    "on this pool's B200 (profiles/r02_i8_peak.txt)")
PEAK_SOURCE = ("measured: DMMA.8x8x4 issue loop on this pool's B200 at 1965 MHz "
               "(profiles/r01_fp64_peak.txt; = 148 SM x 128 flop/clk x 1.965 GHz; "
               "MEASURED_PEAKS.json holds no FP64 figure)")
SEED = 20261019
PROFILE_TAG = "r02"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=100_000, help="SNPs per GPU")
    ap.add_argument("--t", type=int, default=1000)
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--snp-coding", default="genotypes", choices=["genotypes", "real"],
                    help="BASELINE X_R are genotype codes {0,1,2}: exact int8 tcgen05 rotation")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise torch.distributed (NCCL) and run the broadcast / barrier / "
                         "max-over-ranks code even at world size 1 (exercises the multi-GPU "
                         "plumbing on a one-GPU box; needs the torchrun environment)")
    ap.add_argument("--no-alt-coding", dest="alt_coding", action="store_false",
                    help="skip timing the other SNP coding on the same data")
    ap.add_argument("--no-cpu", action="store_true",
                    help="skip the CPU baseline (and with it the every-cell parity)")
    ap.add_argument("--layout", default="stream", choices=["numpy", "stream"],
                    help="result order: the reference's compute_tile ResultTile / run_grid "
                         "result-stream order (j*m + i)*p (grid.hpp:129-148, stream.hpp:31-34; "
                         "default), or numpy (m, t, p) as gwgrid.solve_grid reorders it on the host")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="engine option (gwg_set_option), e.g. i8_cluster=2; for A/B timing")
    return ap.parse_args()


class Clocks:
    """Samples SM clock and throttle reasons through NVML (pynvml) on a
    background thread for the duration of the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples, self.reasons, self.max_mhz = [], set(), None

    def _run(self):
        import pynvml

        h = self.handle
        while not self.stop.is_set():
            try:
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop.wait(self.period)

    def __enter__(self):
        import threading

        self.stop = threading.Event()
        self.thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=5)

    def summary(self) -> dict:
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(sm)}




def make_inputs(args, rank: int, world: int, dev_index: int):
    """Shared operands from rank 0 (kinship eig on the CPU), broadcast once by
    multi.broadcast_shared; each rank generates only its own SNP shard
    (weak scaling: global columns [rank m, (rank + 1) m))."""
    import torch

    from paper_1210_7683_b200 import datagen, eigendecompose, multi

    n, p, m, t = args.n, args.p, args.m, args.t
    dev = torch.device("cuda", dev_index)
    shared_np, eig_s = None, None
    if rank == 0:
        phi = datagen.kinship(SEED, n, 2 * n)
        t0 = time.perf_counter()
        basis, values = eigendecompose(phi)
        eig_s = time.perf_counter() - t0
        shared_np = {"basis": basis, "values": values, "xl": datagen.covariates(SEED, n, p),
                     "y": datagen.normals(SEED, datagen.M_TRAITS, n, 0, t),
                     "h2": datagen.uniform(SEED, datagen.M_H2, t, 0.05, 0.95),
                     "sigma2": np.ones(t)}
    shared = multi.broadcast_shared(shared_np, n, p, t, device=dev)
    torch.cuda.synchronize(dev)
    shared["eig_s"] = eig_s
    i0, i1 = multi.rank_range(m * world, world, rank)
    x_host = torch.empty((m, n), dtype=torch.float64).pin_memory()
    xh = x_host.numpy().T  # (n, m) column-major view
    datagen.genotypes(SEED, datagen.M_SNPS, n, i0, i1 - i0, out=xh)
    return shared, x_host, xh, i0


def run_ours(args):
    import torch

    import paper_1210_7683_b200 as gw
    from paper_1210_7683_b200 import multi

    world, rank, local = multi.dist_env()
    use_dist = world > 1 or args.force_dist
    if use_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    n, p, m, t = args.n, args.p, args.m, args.t
    shared, x_host_t, x_host, i0 = make_inputs(args, rank, world, local)
    dev = torch.device("cuda", local)

    eng = gw.Engine(n, p, device=local)
    eng.set_spectrum(shared["basis"], shared["values"])
    eng.set_covariates(shared["xl"])
    eng.set_snp_coding(args.snp_coding)
    for opt in args.option:
        name, value = opt.split("=", 1)
        eng.set_option(name, int(value))
    x_dev = x_host_t.to(dev, non_blocking=False).t()  # (n, m) column-major on device
    shape = (m, t, p) if args.layout == "numpy" else (t, m, p)
    b_dev = torch.empty(shape, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(eng.compute_stream, device=dev)

    def step():
        eng.set_traits(shared["y"], shared["h2"], shared["sigma2"])
        eng.solve_snp_slab(x_dev, out=b_dev, i0=i0, layout=args.layout)

    def barrier():
        if use_dist:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if not use_dist:
            return v
        import torch.distributed as dist

        tm = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        return float(tm.item())

    for _ in range(args.warmup):
        step()
    barrier()
    eng.reset_counters()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        eng.synchronize()  # the steps' error words (device outputs are asynchronous)
        ev1.record(stream)
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    cnt = eng.counters()
    ms_step = max_over_ranks(ms_total) / args.steps
    cells = m * t * world
    value = cells / (ms_step * 1e-3)
    grid_flops_step = m * t * 2 * n * (p + 1)
    kernel_ms = cnt["grid_kernel_ms"] / args.steps
    rotate_ms = cnt["rotate_ms"] / args.steps
    split = cnt["quad_ms"] > 0
    if split:
        # genotype split grid, two tensor-bound stages:
        #  * S_BR on DMMA (gls_sbr_kernel): factorised as ((X'.X')^T E) F with r
        #    exponential-sum terms, 2 r (n + t) flop per SNP (or the direct
        #    contraction, 2 n flop per cell, when sbr_terms = 0);
        #  * linear_solve_kernel: the p linear terms exactly on the int8 tensor
        #    cores (7 slices of W, 2 n p ops per slice per cell) + the solve.
        # The primary roofline entry is the stage with the larger share.
        quad_ms = cnt["quad_ms"] / args.steps
        lin_ms = cnt["linear_ms"] / args.steps
        r_terms = int(cnt["sbr_terms"])
        quad_flops = cnt["sbr_flops"] // args.steps
        achieved = quad_flops / (quad_ms * 1e-3) / 1e12
        lin_ops = m * t * p * 2 * n * I8_SLICES
        lin_achieved = lin_ops / (lin_ms * 1e-3) / 1e12
        sbr_entry = {"bound": "tensor", "achieved": achieved, "peak": PEAK_FP64_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / PEAK_FP64_TFLOPS,
                     "traffic": load_traffic("sbr_kernel"),
                     "kernel": ("gls_sbr_kernel x2 (G = (X'.X')^T E, S_BR = G F; r = %d)" % r_terms
                                if r_terms else "gls_sbr_kernel"),
                     "kernel_ms": quad_ms, "peak_source": PEAK_SOURCE,
                     "algorithmic_flops_per_launch": quad_flops,
                     "algorithmic_unit": ("2 r (n + t) flop per SNP: S_BR = ((X'.X')^T E) F"
                                          if r_terms else "2n flop per cell: S_BR = (X'.X')^T D")}
        lin_entry = {"bound": "tensor", "achieved": lin_achieved, "peak": PEAK_INT8_TOPS,
                     "unit": "TOP/s", "frac": lin_achieved / PEAK_INT8_TOPS,
                     "traffic": load_traffic("linear_solve_kernel"),
                     "kernel": "linear_solve_kernel<P=%d> (x^T W on 7 int8 slices + bordered "
                               "Cholesky)" % p,
                     "kernel_ms": lin_ms, "peak_source": PEAK_INT8_SOURCE,
                     "algorithmic_ops_per_launch": lin_ops,
                     "algorithmic_unit": "2 n p int8 ops per slice per cell, 7 slices"}
        primary, secondary = (lin_entry, sbr_entry) if lin_ms >= quad_ms else (sbr_entry, lin_entry)
        roof = dict(primary)
        roof["secondary"] = secondary
        roof["grid_fp64_equivalent_tflops"] = grid_flops_step / ((quad_ms + lin_ms) * 1e-3) / 1e12
        roof["step_breakdown_ms"] = {"rotate_snps": rotate_ms, "sbr": quad_ms,
                                     "linear_solve": lin_ms,
                                     "other (Y rotation, contexts, W, E/F)": ms_step - rotate_ms
                                     - lin_ms - quad_ms}
    else:
        # all-FP64 path: the grid launch group is the S_BR stage (factorised,
        # when sbr_flops > 0) + the grid kernel (2np flop per cell then; the
        # fused 2n(p+1) otherwise); achieved = the flops it actually issues
        sbr_step = cnt["sbr_flops"] // args.steps
        issued = (m * t * 2 * n * p + sbr_step) if sbr_step else grid_flops_step
        achieved = issued / (kernel_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": PEAK_FP64_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / PEAK_FP64_TFLOPS,
                "traffic": load_traffic("grid_kernel") if not sbr_step else None,
                "kernel": ("gls_sbr_kernel x2 + gls_grid_kernel<P=%d, EXT> (S_BR factorised, r = %d)"
                           % (p, cnt["sbr_terms"]) if sbr_step else "gls_grid_kernel<P=%d>" % p),
                "kernel_ms": kernel_ms, "rotate_ms": rotate_ms, "peak_source": PEAK_SOURCE,
                "algorithmic_flops_per_launch": issued,
                "grid_fp64_equivalent_tflops": grid_flops_step / (kernel_ms * 1e-3) / 1e12}

    bad = int(torch.isnan(b_dev).sum().item())

    # ---- the other SNP coding on the same data, for transparency: the all-FP64
    # path (real coding) when the headline runs the genotype path -------------
    alt = None
    if args.alt_coding:
        other = "real" if args.snp_coding == "genotypes" else "genotypes"
        eng.set_snp_coding(other)
        b_alt = torch.empty_like(b_dev)

        def alt_step():
            eng.set_traits(shared["y"], shared["h2"], shared["sigma2"])
            eng.solve_snp_slab(x_dev, out=b_alt, i0=i0, layout=args.layout)

        alt_step()
        barrier()
        eng.reset_counters()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            alt_step()
        eng.synchronize()
        a1.record(stream)
        barrier()
        alt_ms = a0.elapsed_time(a1) / args.steps
        acnt = eng.counters()
        rel = ((b_alt - b_dev).norm(dim=-1) / b_dev.norm(dim=-1)).max().item()
        alt = {"snp_coding": other, "value": cells / (alt_ms * 1e-3), "ms_per_step": alt_ms,
               "grid_kernel_ms": acnt["grid_kernel_ms"] / args.steps,
               "max_normwise_rel_diff_vs_headline": rel}
        eng.set_snp_coding(args.snp_coding)
        del b_alt

    # ---- e2e through gwg_set_traits + gwg_run_grid with pinned host buffers --
    e2e = e2e_i8 = None
    if not args.no_e2e:
        # e2e returns b the way gwgrid.solve_grid does, (m, t, p) in host
        # memory: one contiguous D2H run per slab (the stream order would
        # need a strided 2-D copy, measured slower over PCIe)
        b_host_t = torch.empty((m, t, p), dtype=torch.float64).pin_memory()
        b_host = b_host_t.numpy()
        y_host_t = torch.empty((t, n), dtype=torch.float64).pin_memory()
        y_host_t.copy_(shared["y"].t())
        y_host = y_host_t.numpy().T
        h2_host = shared["h2"].cpu().numpy()
        s2_host = np.ones(t)
        codes_t = torch.empty((m, n), dtype=torch.int8).pin_memory()
        codes_t.copy_(x_host_t.to(torch.int8))
        codes = codes_t.numpy().T  # (n, m) int8, column-major, pinned

        def timed_e2e(snps):
            def e2e_step():
                eng.set_traits(y_host, h2_host, s2_host)
                eng.run_grid(snps, out=b_host, i0=i0, layout="numpy")

            for _ in range(max(1, args.warmup - 1)):
                e2e_step()
            barrier()
            eng.reset_counters()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                e2e_step()
            barrier()
            e2e_s = max_over_ranks(time.perf_counter() - t0)
            dv = b_dev.cpu().numpy()
            same = bool(np.array_equal(b_host, dv if args.layout == "numpy" else dv.transpose(1, 0, 2)))
            c = eng.counters()
            return e2e_s, same, c

        e2e_s, same, c = timed_e2e(x_host)
        e2e = {"value": cells * args.steps / e2e_s, "unit": "GLS/s",
               "h2d_bytes_per_step": n * m * 8 + n * t * 8 + 2 * t * 8,
               "d2h_bytes_per_step": m * t * p * 8, "ms_per_step": 1e3 * e2e_s / args.steps,
               "io_stall_ms_per_step": c["io_stall_ms"] / args.steps,
               "api": "Engine.set_traits + Engine.run_grid (gwg_set_traits + gwg_run_grid), "
                      "X_R as float64 (BASELINE's storage), b returned as (m, t, p) like "
                      "gwgrid.solve_grid",
               "bitwise_equal_to_device_path": same}
        e2e_s, same, c = timed_e2e(codes)
        e2e_i8 = {"value": cells * args.steps / e2e_s, "unit": "GLS/s",
                  "h2d_bytes_per_step": n * m + n * t * 8 + 2 * t * 8,
                  "d2h_bytes_per_step": m * t * p * 8, "ms_per_step": 1e3 * e2e_s / args.steps,
                  "io_stall_ms_per_step": c["io_stall_ms"] / args.steps,
                  "api": "the same with X_R as int8 genotype codes (GWG_FORMAT_I8)",
                  "bitwise_equal_to_device_path": same}
        del b_host_t, codes_t

    # ---- CPU baseline (oracle) on the full grid, and every-cell parity -------
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.parity import parity_metrics

        cpu, ref = cpu_baseline(args, shared, x_host)
        got = b_dev.cpu().numpy()
        got = got if args.layout == "numpy" else got.transpose(1, 0, 2)
        parity = parity_metrics(got, ref)
        del ref
        parity["vs_reference_build"] = parity_vs_reference_build(args, shared, x_host, got)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GLS/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE.json generators, seed %d)" % SEED,
            "config": {"workload": "c1", "n": n, "p": p, "m_per_gpu": m, "t": t,
                       "cells_per_step": cells, "parallelism": f"snp-shard x{world}",
                       "l2": "inputs larger than L2 (X_R %.1f GB per GPU per step)" % (n * m * 8 / 1e9),
                       "snp_coding": args.snp_coding, "result_layout": args.layout,
                       "step": ("rotate Y (DMMA) and X_R (exact int8 tcgen05) + trait contexts "
                                "+ split grid: S_BR = (X'.X')^T D on DMMA, linear terms x^T W exact "
                                "on int8 tcgen05 fused with the bordered Cholesky"
                                if split else
                                "rotate Y and X_R (DMMA) + trait contexts + fused DMMA grid kernel")},
            "tflops": grid_flops_step * world / (ms_step * 1e-3) / 1e12,
            "tflops_convention": "2n(p+1) per cell (grid contraction); reference n(2p+3) = %.3f TF"
                                 % (m * t * n * (2 * p + 3) * world / (ms_step * 1e-3) / 1e12),
            "gpu_launches": int(cnt["kernel_launches"]),
            "roofline": roof,
            "clocks": clk.summary(),
            "e2e": e2e,
            "e2e_int8": e2e_i8,
            "cpu_baseline": cpu,
            "parity": parity,
            "nan_cells": bad,
            "other_coding": alt,
            "preloop_eig_s": shared.get("eig_s"),
        }
        if args.option:
            line["config"]["engine_options"] = args.option
        print(json.dumps(line), flush=True)
    eng.close()
    if use_dist:
        import torch.distributed as dist

        dist.destroy_process_group()


def load_traffic(name: str):
    for tag in (PROFILE_TAG, "r01"):
        path = os.path.join(ROOT, "profiles", "%s_%s_ncu.json" % (tag, name))
        try:
            with open(path) as f:
                return json.load(f).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            continue
    return None


def cpu_sample_run(basis, values, xl, y, h2, x_sample, workers):
    """The reference CPU step: OpenBLAS rotations + contexts + compute_tile
    (CT, 160x160 blocks, `workers` threads) — oracle/ (test infrastructure)."""
    from oracle import oracle as orc

    orc.set_blas_threads(workers)
    xr = orc.rotate(basis, x_sample)
    yr = orc.rotate(basis, y)
    xlr = orc.rotate(basis, xl)
    return orc.compute_grid(values, xlr, xr, yr, h2, np.ones(len(h2)), workers=workers)


def cpu_baseline(args, shared, x_host):
    """The oracle's reference CPU step over the SAME full grid the device just
    timed (rank 0, N = 1): its time is the cpu_baseline, its grid the parity
    reference."""
    basis = shared["basis"].cpu().numpy()
    values = shared["values"].cpu().numpy()
    xl = shared["xl"].cpu().numpy()
    y = shared["y"].cpu().numpy()
    h2 = shared["h2"].cpu().numpy()
    workers = os.cpu_count() or 1
    xs = np.asfortranarray(x_host)
    cpu_sample_run(basis, values, xl, y, h2, xs[:, :160], workers)  # warm
    t0 = time.perf_counter()
    ref = cpu_sample_run(basis, values, xl, y, h2, xs, workers)
    dt = time.perf_counter() - t0
    ms = xs.shape[1]
    return ({"value": ms * args.t / dt, "unit": "GLS/s", "cores": workers, "kind": "port",
             "sample": f"the full c1 grid: {ms} SNPs x {args.t} traits (rotation + contexts + "
                       f"compute_tile CT, {workers} worker threads, OpenBLAS {workers} threads), "
                       f"{dt:.1f} s"}, ref)


def run_reference(args):
    """bench.py --impl reference: the reference's CPU path (oracle/, the
    restated gwgrid compute_tile CT scheduler + OpenBLAS rotation) over the
    same full c1 grid per step.  Inputs come from the oracle library's own
    copy of the seeded generator; no engine library is loaded."""
    from paper_1210_7683_b200 import multi

    world, rank, _ = multi.dist_env()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_1210_7683_b200 import datagen  # pure Python; generator calls go to `lib`

    lib = orc.load()
    n, p, m, t = args.n, args.p, args.m, args.t
    phi = datagen.kinship(SEED, n, 2 * n, lib=lib)
    basis, values = orc.eigendecompose(phi)
    xl = datagen.covariates(SEED, n, p, lib=lib)
    y = datagen.normals(SEED, datagen.M_TRAITS, n, 0, t, lib=lib)
    h2 = datagen.uniform(SEED, datagen.M_H2, t, 0.05, 0.95, lib=lib)
    xs = datagen.genotypes(SEED, datagen.M_SNPS, n, 0, m, lib=lib)
    workers = os.cpu_count() or 1
    warm = min(m, 2000)
    for _ in range(args.warmup):  # BLAS threads and caches: a 2,000-SNP slice
        cpu_sample_run(basis, values, xl, y, h2, xs[:, :warm], workers)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_sample_run(basis, values, xl, y, h2, xs, workers)
    dt = (time.perf_counter() - t0) / args.steps
    value = m * t / dt
    ref_build = reference_build_sample(basis, values, xl, y, h2, xs, workers)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GLS/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json generators, seed %d)" % SEED,
        "config": {"workload": "c1", "n": n, "p": p, "m_per_gpu": m, "t": t,
                   "cells_per_step": m * t,
                   "parallelism": "host threads x%d (rank 0)" % workers,
                   "snp_coding": "real (the reference's double-precision CPU path)",
                   "warmup_sample": f"{warm} SNPs x {t} traits"},
        "cpu_baseline": {"value": value, "unit": "GLS/s", "cores": workers, "kind": "port",
                         "sample": f"the full c1 grid per step: {m} SNPs x {t} traits (oracle/ "
                                   "restatement of gwgrid compute_tile CT + OpenBLAS rotation)"},
        "e2e": {"value": value, "unit": "GLS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_build": ref_build,
        "note": "value = the oracle/ C++ restatement of gwgrid's CPU path (the faster of the two "
                "CPU implementations here, so the conservative baseline); reference_build = "
                "gwgrid's own gls.cpp/grid.cpp compiled in place against our Eigen stand-in "
                "(Eigen3 is absent from the image; oracle/refbuild), timed on a bounded sample; "
                "inputs from the oracle library's copy of the generator (no engine code loaded)",
    }
    print(json.dumps(line), flush=True)


def parity_vs_reference_build(args, shared, x_host, got, slab=20_000):
    """The timed device grid, EVERY cell, against the REFERENCE'S OWN sources
    (oracle/_ref/libgwgrid_ref.so: gwgrid's rotate_columns + build_trait_contexts
    + compute_tile CT, compiled in place against the Eigen stand-in) run on the
    host cores in slabs of `slab` SNPs, when the prebuilt library is present
    (test infrastructure; never on the product path)."""
    from oracle import ref
    from oracle.parity import parity_metrics

    if not os.path.exists(ref.LIB_PATH):
        return {"unavailable": "oracle/_ref/libgwgrid_ref.so not present"}
    m = x_host.shape[1]
    h2 = shared["h2"].cpu().numpy()
    basis, values = shared["basis"].cpu().numpy(), shared["values"].cpu().numpy()
    xl, y = shared["xl"].cpu().numpy(), shared["y"].cpu().numpy()
    workers = os.cpu_count() or 1
    out = {"cells": 0, "components": 0, "normwise_max": 0.0, "floored_componentwise_max": 0.0,
           "floored5_componentwise_max": 0.0, "raw_componentwise_max": 0.0,
           "n_floored_over_1e-8": 0, "n_raw_over_1e-8": 0, "pass": True}
    t0 = time.perf_counter()
    for i0 in range(0, m, slab):
        want = ref.compute_grid(basis, values, xl, np.asfortranarray(x_host[:, i0:i0 + slab]), y,
                                h2, np.ones(len(h2)), workers=workers)
        pm = parity_metrics(np.ascontiguousarray(got[i0:i0 + slab]), want)
        del want
        for k in out:
            if k == "pass":
                out[k] = bool(out[k] and pm[k])
            elif k.endswith("_max"):
                out[k] = max(out[k], pm[k])
            else:
                out[k] += pm[k]
    out["tolerance"] = pm["tolerance"]
    out["reference"] = ("gwgrid's own rotate_columns + build_trait_contexts + compute_tile "
                        f"(oracle/_ref), all {m} SNPs x {len(h2)} traits in slabs of {slab}, "
                        f"{time.perf_counter() - t0:.0f} s on {workers} host threads")
    return out


def reference_build_sample(basis, values, xl, y, h2, xs, workers, sample=10_000):
    """The reference's OWN sources (oracle/_ref/libgwgrid_ref.so: gwgrid's
    rotate_columns + build_trait_contexts + compute_tile CT, compiled against
    the Eigen stand-in) on a bounded sample of the same grid, when the prebuilt
    library is present; its grid is compared with the restatement's."""
    from oracle import ref

    if not os.path.exists(ref.LIB_PATH):
        return {"unavailable": "oracle/_ref/libgwgrid_ref.so not present"}
    ms = min(sample, xs.shape[1])
    sub = np.asfortranarray(xs[:, :ms])
    s2 = np.ones(len(h2))
    ref.compute_grid(basis, values, xl, sub[:, :min(ms, 500)], y, h2, s2, workers=workers)  # warm
    t0 = time.perf_counter()
    got = ref.compute_grid(basis, values, xl, sub, y, h2, s2, workers=workers)
    dt = time.perf_counter() - t0
    port = cpu_sample_run(basis, values, xl, y, h2, sub, workers)
    rel = np.linalg.norm(got - port, axis=2) / np.linalg.norm(port, axis=2)
    return {"value": ms * len(h2) / dt, "unit": "GLS/s", "cores": workers, "kind": "reference",
            "sample": f"{ms} SNPs x {len(h2)} traits of the same grid, {dt:.1f} s",
            "normwise_max_vs_restatement": float(rel.max())}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
