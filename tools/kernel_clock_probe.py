"""SM clock DURING the c1 step's kernels (measurement tool, run under gpurun).

A one-warp probe kernel (tools/clock_probe.cu) co-resident on one SM samples
(globaltimer, clock64) every 20 us while 12 bench steps run back to back on the
engine's stream; a stamp kernel after every step gives the step boundaries, and
the engine's own per-group CUDA-event times (rotation / S_BR / linear_solve)
place the three big kernels inside each step (linear_solve is the last launch of
a step, the two S_BR GEMMs precede it, the int8 rotation precedes those).
Prints the mean SM clock in each window: nvidia-smi's clocks.sm reads 1965 MHz
throughout, ncu's sm__cycles_elapsed.avg.per_second reads ~1.75 GHz for the
int8 kernels; this is the direct measurement.

  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC \
       -o tools/libclock_probe.so tools/clock_probe.cu
  python tools/kernel_clock_probe.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1210_7683_b200 as gw  # noqa: E402
from paper_1210_7683_b200 import datagen  # noqa: E402

STEPS, INTERVAL_NS = 12, 20_000


def main():
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libclock_probe.so"))
    lib.clock_probe_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint]
    lib.clock_stamp_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    n, p, m, t = 1000, 4, 100_000, 1000
    dev = torch.device("cuda", 0)
    ds = datagen.generate(n, p, 8, t, seed=20261019)
    basis, values = gw.eigendecompose(ds["kinship"])
    xh = torch.empty((m, n), dtype=torch.float64).pin_memory()
    datagen.genotypes(20261019, datagen.M_SNPS, n, 0, m, out=xh.numpy().T)
    x_dev = xh.to(dev).t()
    y = torch.from_numpy(np.ascontiguousarray(ds["traits"].T)).to(dev).t()
    h2 = torch.from_numpy(ds["h2"]).to(dev)
    s2 = torch.from_numpy(ds["sigma2"]).to(dev)
    b_dev = torch.empty((t, m, p), dtype=torch.float64, device=dev)
    with gw.Engine(n, p, device=0) as eng:
        eng.set_spectrum(basis, values)
        eng.set_covariates(ds["xl"])
        eng.set_snp_coding("genotypes")

        def step():
            eng.set_traits(y, h2, s2)
            eng.solve_snp_slab(x_dev, out=b_dev, i0=0, layout="stream")

        for _ in range(5):
            step()
        eng.synchronize()
        torch.cuda.synchronize()
        eng.reset_counters()
        nsamp = int(STEPS * 4.6e6 / INTERVAL_NS)
        samples = torch.zeros(2 * nsamp, dtype=torch.int64, device=dev)
        stamps = torch.zeros(STEPS + 1, dtype=torch.int64, device=dev)
        side = torch.cuda.Stream(device=dev)
        torch.cuda.synchronize()
        comp = ctypes.c_void_p(eng.compute_stream)
        # load both tool kernels first (a lazy module load waits for running kernels)
        assert lib.clock_stamp_launch(comp, ctypes.c_void_p(stamps.data_ptr())) == 0
        assert lib.clock_probe_launch(ctypes.c_void_p(side.cuda_stream),
                                      ctypes.c_void_p(samples.data_ptr()), 2, 1000) == 0
        torch.cuda.synchronize()
        assert lib.clock_probe_launch(ctypes.c_void_p(side.cuda_stream), ctypes.c_void_p(samples.data_ptr()),
                                      nsamp, INTERVAL_NS) == 0
        assert lib.clock_stamp_launch(comp, ctypes.c_void_p(stamps.data_ptr())) == 0
        for k in range(STEPS):
            step()
            assert lib.clock_stamp_launch(comp, ctypes.c_void_p(stamps[k + 1:].data_ptr())) == 0
        eng.synchronize()
        torch.cuda.synchronize()
        c = eng.counters()
    s = samples.cpu().numpy().reshape(-1, 2).astype(np.float64)
    st = stamps.cpu().numpy().astype(np.float64)
    tt, cc = s[:, 0], s[:, 1]
    rot_ms = c["rotate_ms"] / STEPS
    lin_ms, sbr_ms = c["linear_ms"] / STEPS, c["quad_ms"] / STEPS

    def mhz(t0, t1):
        i0, i1 = np.searchsorted(tt, t0), np.searchsorted(tt, t1) - 1
        if i1 <= i0:
            return None
        return float((cc[i1] - cc[i0]) / (tt[i1] - tt[i0]) * 1e3)

    gaps = np.diff(tt)
    print("samples", len(tt), "zero", int((tt == 0).sum()), "gap us: median", np.median(gaps) / 1e3,
          "max", gaps.max() / 1e3, "n gaps > 100us", int((gaps > 1e5).sum()), file=sys.stderr)
    print("first stamp - first sample (us)", (st[0] - tt[0]) / 1e3, "last sample - last stamp (us)",
          (tt[-1] - st[-1]) / 1e3, file=sys.stderr)
    big = np.where(gaps > 1e5)[0][:12]
    print("big gaps at (us since first stamp, length us):",
          [(round((tt[i] - st[0]) / 1e3), round(gaps[i] / 1e3)) for i in big], file=sys.stderr)
    rows = []
    for k in range(2, STEPS):
        end = st[k + 1]
        lin0 = end - lin_ms * 1e6
        sbr0 = lin0 - sbr_ms * 1e6
        rot0 = sbr0 - rot_ms * 1e6
        rows.append({"step_ms": (st[k + 1] - st[k]) / 1e6, "linear_mhz": mhz(lin0, end),
                     "sbr_mhz": mhz(sbr0, lin0), "rotate_mhz": mhz(rot0, sbr0),
                     "whole_step_mhz": mhz(st[k], end)})
    med = {key: float(np.median([r[key] for r in rows if r[key] is not None])) for key in rows[0]}
    print(json.dumps({"workload": "c1 device step, genotype path, 12 steps back to back",
                      "per_group_ms": {"rotate": rot_ms, "sbr": sbr_ms, "linear_solve": lin_ms},
                      "median": med, "steps": rows,
                      "idle_before_mhz": mhz(tt[0], st[0])}))


if __name__ == "__main__":
    main()
