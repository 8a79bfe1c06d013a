"""Host-side mirror of the reference gwgrid API over the device engine.

Python face of include/gwgrid_cuda.h.  Names, argument meaning and error
behaviour follow the reference's Python module (proj/python/bindings.cpp and
proj/python/gwgrid/__init__.py):

* ``eigendecompose(phi)``          -> eigendecompose_kinship (gls.cpp:16-46), CPU/LAPACK
* ``solve_grid(kinship, xl, snps, traits, h2, sigma2, ...)``
                                   -> solve_grid_py (bindings.cpp:115-190)
* ``solve_cell(phi, xl, xr, y, h2, sigma2)``
                                   -> solve_partitioned_gls (gls.cpp:162-186)
* ``Engine``                       -> GridPrecompute + build_trait_contexts +
                                      compute_tile / run_grid (grid.hpp:81-237)
* ``Group``                        -> run_grid's worker parallelism
                                      (grid.cpp:519-639) at GPU granularity

Everything after the one-off eigendecomposition runs on the B200 through the
native library; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import time
from typing import Any

import numpy as np

from . import _native as nat
from .errors import DimensionError, InfeasibleBudgetError, NonSymmetricError, raise_for


def _is_torch(x: Any) -> bool:
    return type(x).__module__.split(".")[0] == "torch"


class _Operand:
    """A column-major FP64 operand: host (numpy) or device (torch CUDA).

    A CUDA tensor must live on ``device`` (the engine's GPU).  Instead of a
    host-side synchronize, the engine's stream is ordered after torch's
    current stream on that device (``gwg_wait_stream``) by the caller, who
    also keeps ``keep`` alive until the engine's next synchronising call."""

    def __init__(self, x: Any, shape: tuple, name: str, device: int | None = None):
        self.keep = None
        self.stream = None
        if _is_torch(x):
            import torch

            if x.dtype != torch.float64:
                raise DimensionError(f"{name} must be float64, got {x.dtype}")
            if tuple(x.shape) != tuple(shape):
                raise DimensionError(f"{name} has shape {tuple(x.shape)}, expected {shape}")
            if x.is_cuda and device is not None and x.device.index != device:
                raise DimensionError(f"{name} lives on {x.device}, the engine on cuda:{device}")
            if x.dim() == 2 and x.shape[0] > 1 and x.shape[1] > 1 and not (
                    x.stride(0) == 1 and x.stride(1) == x.shape[0]):
                x = x.t().contiguous().t()
            elif x.dim() <= 1 or x.shape[0] <= 1 or x.shape[1] <= 1:
                x = x.contiguous()
            if x.is_cuda:
                if device is None:  # no engine stream to order: wait on the host
                    torch.cuda.current_stream(x.device).synchronize()
                else:
                    self.stream = torch.cuda.current_stream(x.device).cuda_stream
            self.keep = x
            self.ptr = x.data_ptr()
            self.where = nat.GWG_DEVICE if x.is_cuda else nat.GWG_HOST
        else:
            a = np.asarray(x, dtype=np.float64)
            if a.shape != tuple(shape):
                raise DimensionError(f"{name} has shape {a.shape}, expected {shape}")
            a = np.asfortranarray(a)
            self.keep = a
            self.ptr = a.ctypes.data
            self.where = nat.GWG_HOST


def eigendecompose(phi: np.ndarray, device: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Kinship eigensystem with the reference's contract (gls.cpp:16-46).

    Symmetry gate max|Phi - Phi^T| <= 1e-12 max|Phi|; ascending eigenvalues;
    each eigenvector's largest-magnitude entry (first on ties) made positive.
    By default on the CPU (LAPACK dsyevd via numpy), as the north star keeps
    it; ``device=k`` runs it on GPU k (cuSOLVER syevd + this library's gate
    and sign-rule kernels, gwg_eigendecompose).
    """
    if device is not None:
        lib = nat.load()
        a = np.asfortranarray(np.asarray(phi, dtype=np.float64))
        if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
            raise DimensionError("relatedness matrix must be square and non-empty")
        n = a.shape[0]
        basis = np.empty((n, n), dtype=np.float64, order="F")
        values = np.empty(n, dtype=np.float64)
        st = nat.Status()
        rc = lib.gwg_eigendecompose(int(device), n, a.ctypes.data, nat.GWG_HOST,
                                    basis.ctypes.data, values.ctypes.data, nat.GWG_HOST,
                                    ctypes.byref(st))
        if rc != nat.GWG_OK:
            raise_for(st)
        return basis, values
    phi = np.asarray(phi, dtype=np.float64)
    if phi.ndim != 2 or phi.shape[0] != phi.shape[1] or phi.shape[0] < 1:
        raise DimensionError("relatedness matrix must be square and non-empty")
    scale = float(np.max(np.abs(phi)))
    asym = float(np.max(np.abs(phi - phi.T)))
    if asym > 1e-12 * scale:
        raise NonSymmetricError(
            f"relatedness matrix is not symmetric: max|A-A'|={asym:g} exceeds "
            f"1e-12*max|A|={1e-12 * scale:g}")
    values, basis = np.linalg.eigh(phi, UPLO="L")
    idx = np.argmax(np.abs(basis), axis=0)
    signs = np.where(basis[idx, np.arange(basis.shape[1])] < 0.0, -1.0, 1.0)
    basis = np.asfortranarray(basis * signs)
    return basis, values


def _snp_array(snps, n: int):
    """(n, m) SNP operand for run_grid: int8 genotype codes stay int8
    (GWG_FORMAT_I8, 1 byte per code), anything else becomes float64."""
    snps = np.asarray(snps)
    fmt = nat.GWG_FORMAT_I8 if snps.dtype == np.int8 else nat.GWG_FORMAT_F64
    if fmt == nat.GWG_FORMAT_F64:
        snps = snps.astype(np.float64, copy=False)
    snps = np.asfortranarray(snps)
    if snps.ndim != 2 or snps.shape[0] != n:
        raise DimensionError(f"snps must be (n={n}, m), got {snps.shape}")
    return snps, fmt


def _run_options(t: int, p: int, m: int, layout: str, mb: int, double_buffer: bool,
                 checksum: bool, i0: int, sink, ring: int, ldb: int, fmt: int, out):
    """gwg_run_options + the output buffer (or the sink trampoline) of a
    run_grid call; returns (opts, out, out_ptr, keep, errors)."""
    lay = nat.GWG_LAYOUT_NUMPY if layout == "numpy" else nat.GWG_LAYOUT_STREAM
    if layout not in ("numpy", "stream"):
        raise DimensionError(f"unknown layout {layout!r}")
    opts = nat.RunOptions()
    opts.mb, opts.layout, opts.double_buffer = int(mb), lay, int(bool(double_buffer))
    opts.snp_format, opts.checksum, opts.i0 = fmt, int(bool(checksum)), int(i0)
    opts.ring, opts.ldb = int(ring), int(ldb)
    errors: list = []
    keep = None
    if sink is not None:
        def trampoline(_user, gi0, rows, ptr):
            try:
                shape = (rows, t, p) if lay == nat.GWG_LAYOUT_NUMPY else (t, rows, p)
                cells = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)),
                                              shape=shape)
                sink(int(gi0), cells)
                return 0
            except BaseException as exc:  # noqa: BLE001 - re-raised by the caller
                errors.append(exc)
                return 1

        keep = nat.RESULT_SINK(trampoline)
        opts.sink = keep
        return opts, None, None, keep, errors
    rows_b = max(int(ldb), m)
    shape = (m, t, p) if lay == nat.GWG_LAYOUT_NUMPY else (t, rows_b, p)
    if out is None:
        out = np.empty(shape, dtype=np.float64)
    if out.shape != shape or not out.flags.c_contiguous or out.dtype != np.float64:
        raise DimensionError(f"out must be a C-contiguous float64 array of shape {shape}")
    return opts, out, out.ctypes.data, keep, errors


class Engine:
    """One device engine: spectrum + covariates + traits resident in HBM.

    Calls on one Engine must be serialised (one host thread per GPU), like the
    reference's CT coordinator (grid.cpp:519-552).
    """

    def __init__(self, n: int, p: int, device: int = 0, _handle: int | None = None):
        self._lib = nat.load()
        self.n, self.p, self.t = int(n), int(p), 0
        self.device = int(device)
        self._owned = _handle is None
        if _handle is not None:  # an engine owned by a Group
            self._h = _handle
        else:
            st = nat.Status()
            self._h = self._lib.gwg_engine_create(self.device, self.n, self.p, ctypes.byref(st))
            if not self._h:
                raise_for(st)
                raise DimensionError("engine creation failed")
        # device operands of queued (not yet synchronised) work stay referenced
        self._pending: list = []

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            if self._owned:
                self._lib.gwg_engine_destroy(self._h)
            self._h = None
            self._pending = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, fn, *args) -> None:
        st = nat.Status()
        rc = fn(self._h, *args, ctypes.byref(st))
        if rc != nat.GWG_OK:
            raise_for(st)

    def _operand(self, x, shape, name) -> _Operand:
        """Wrap an operand; a torch CUDA tensor orders the engine's stream
        after torch's (no host round trip) and stays referenced until the
        engine next synchronises."""
        op = _Operand(x, shape, name, device=self.device)
        if op.stream is not None:
            self._call(self._lib.gwg_wait_stream, op.stream)
            self._pending.append(op.keep)
        return op

    def _synced(self) -> None:
        self._pending = []

    # -- options -----------------------------------------------------------
    def set_option(self, name: str, value: int) -> None:
        """gwg_set_option: "split", "sbr_direct", "real_split", "i8_cluster",
        "sbr_cfg" (include/gwgrid_cuda.h)."""
        if name not in nat.OPTIONS:
            raise DimensionError(f"unknown option {name!r}")
        self._call(self._lib.gwg_set_option, nat.OPTIONS[name], int(value))

    def get_option(self, name: str) -> int:
        if name not in nat.OPTIONS:
            raise DimensionError(f"unknown option {name!r}")
        v = ctypes.c_int64()
        self._call(self._lib.gwg_get_option, nat.OPTIONS[name], ctypes.byref(v))
        return int(v.value)

    # -- operands ----------------------------------------------------------
    def set_spectrum(self, basis, values) -> None:
        b = self._operand(basis, (self.n, self.n), "basis")
        v = self._operand(values, (self.n,), "values")
        if b.where != v.where:
            raise DimensionError("basis and values must live on the same side")
        self._call(self._lib.gwg_set_spectrum, b.ptr, v.ptr, b.where)
        self._synced()  # the spectrum's range is read back: the stream is drained

    def set_kinship(self, phi) -> None:
        """Eigendecompose phi on the device and install the spectrum
        (gwg_set_kinship; the basis never visits the host)."""
        k = self._operand(phi, (self.n, self.n), "kinship")
        self._call(self._lib.gwg_set_kinship, k.ptr, k.where)
        self._synced()

    def set_snp_coding(self, coding: str) -> None:
        """"auto" (default: per slab, the exact int8 genotype path when every
        value is an integer code in [-127, 127], else the FP64 path), "real"
        (any SNP values, DMMA rotation and grid) or "genotypes" (integer codes
        required, checked on the device) — gwg_set_snp_coding."""
        code = {"real": nat.GWG_SNP_REAL, "genotypes": nat.GWG_SNP_GENOTYPES,
                "auto": nat.GWG_SNP_AUTO}.get(coding)
        if code is None:
            raise DimensionError(f"unknown SNP coding {coding!r}")
        self._call(self._lib.gwg_set_snp_coding, code)

    def set_covariates(self, xl) -> None:
        if self.p == 1:
            self._call(self._lib.gwg_set_covariates, None, nat.GWG_HOST)
            return
        x = self._operand(xl, (self.n, self.p - 1), "xl")
        self._call(self._lib.gwg_set_covariates, x.ptr, x.where)

    def set_traits(self, traits, h2, sigma2, rotated: bool = False) -> None:
        """transform_trait_slab + build_trait_contexts on the device.  Device
        (torch CUDA) operands make this asynchronous; a trait failing the
        weight floor is raised by the next solve_snp_slab / run_grid /
        synchronize (NotPositiveDefiniteError with snp_index -1)."""
        t = int(np.shape(traits)[1]) if np.ndim(traits) == 2 else 1
        y = self._operand(traits if np.ndim(traits) == 2 else np.reshape(traits, (-1, 1)),
                          (self.n, t), "traits")
        h = self._operand(h2, (t,), "h2")
        s = self._operand(sigma2, (t,), "sigma2")
        if not (y.where == h.where == s.where):
            raise DimensionError("traits, h2 and sigma2 must live on the same side")
        self._call(self._lib.gwg_set_traits, t, y.ptr, h.ptr, s.ptr, y.where, int(rotated))
        self.t = t

    # -- grid --------------------------------------------------------------
    def solve_snp_slab(self, x_r, out=None, i0: int = 0, rotated: bool = False,
                       layout: str = "numpy"):
        """compute_tile for one SNP slab against every installed trait.

        Returns ``out``: (mb, t, p) for layout "numpy"; (t, mb, p) for
        "stream" (the GWG1 result order (j*m + i)*p).  A torch CUDA ``out``
        (float64, on the engine's device) keeps the results on the device
        and makes the call asynchronous, like the device work itself: it
        returns once the work is queued on the engine's stream (torch's
        stream.synchronize or torch.cuda.synchronize waits for it), and a
        failing cell or trait is raised by the next synchronising call
        (synchronize, a host-output solve, run_grid) with its coordinates.
        """
        mb = int(np.shape(x_r)[1])
        x = self._operand(x_r, (self.n, mb), "snps")
        lay = nat.GWG_LAYOUT_NUMPY if layout == "numpy" else nat.GWG_LAYOUT_STREAM
        shape = (mb, self.t, self.p) if lay == nat.GWG_LAYOUT_NUMPY else (self.t, mb, self.p)
        if out is None:
            out = np.empty(shape, dtype=np.float64)
        if _is_torch(out):
            import torch

            if out.dtype != torch.float64:
                raise DimensionError(f"out must be float64, got {out.dtype}")
            if tuple(out.shape) != shape or not out.is_contiguous():
                raise DimensionError(f"out must be a contiguous tensor of shape {shape}")
            if out.is_cuda:
                if out.device.index != self.device:
                    raise DimensionError(f"out lives on {out.device}, the engine on "
                                         f"cuda:{self.device}")
                # torch work still using `out` finishes before the engine writes it
                self._call(self._lib.gwg_wait_stream,
                           torch.cuda.current_stream(out.device).cuda_stream)
            optr, owhere = out.data_ptr(), nat.GWG_DEVICE if out.is_cuda else nat.GWG_HOST
        else:
            if out.shape != shape or not out.flags.c_contiguous or out.dtype != np.float64:
                raise DimensionError(f"out must be a C-contiguous float64 array of shape {shape}")
            optr, owhere = out.ctypes.data, nat.GWG_HOST
        try:
            self._call(self._lib.gwg_solve_snp_slab, int(i0), mb, x.ptr, x.where, int(rotated),
                       optr, owhere, lay, mb)
        except BaseException:
            self._synced()
            raise
        if owhere != nat.GWG_DEVICE:  # synchronous: the operands were consumed
            self._synced()
        elif _is_torch(out):  # torch work queued after this call reads `out` in order
            import torch

            self._call(self._lib.gwg_signal_stream,
                       torch.cuda.current_stream(out.device).cuda_stream)
        return out

    def run_grid(self, snps, out=None, layout: str = "numpy", mb: int = 0,
                 double_buffer: bool = True, checksum: bool = False, i0: int = 0,
                 sink=None, ring: int = 0, ldb: int = 0):
        """Stream the whole grid from host memory (run_grid, grid.cpp:454-641).

        ``snps``: (n, m) float64 (any real values), or int8 genotype codes
        (GWG_FORMAT_I8: 1 byte per code over PCIe).  Results go to ``out``
        ((m, t, p) numpy order / (t, max(ldb, m), p) stream order, allocated
        when None), or, with ``sink``, to ``sink(i0, cells)`` slab by slab —
        ``cells`` a view of a pinned buffer, (rows, t, p) or (t, rows, p),
        valid only during the call, ``i0`` the slab's global first SNP — and
        run_grid returns None.  ``checksum`` accumulates the order-independent
        device checksum into counters()["checksum"]; ``i0`` is the global
        index of snps' first column (a shard of a larger grid)."""
        snps, fmt = _snp_array(snps, self.n)
        m = snps.shape[1]
        opts, out, out_ptr, keep, errors = _run_options(self.t, self.p, m, layout, mb,
                                                        double_buffer, checksum, i0, sink,
                                                        ring, ldb, fmt, out)
        cnt = nat.Counters()
        st = nat.Status()
        try:
            rc = self._lib.gwg_run_grid(self._h, m, snps.ctypes.data, out_ptr, ctypes.byref(opts),
                                        ctypes.byref(cnt), ctypes.byref(st))
        finally:
            self._synced()
        del keep
        if errors:
            raise errors[0]
        if rc != nat.GWG_OK:
            raise_for(st)
        return out

    def set_traits_file(self, path: str) -> None:
        """load_pass from a GWG1 trait stream (kind 2)."""
        self._call(self._lib.gwg_set_traits_file, os.fsencode(path))
        st = nat.Status()
        kind, dims, complete = ctypes.c_int32(), (ctypes.c_int64 * 3)(), ctypes.c_int32()
        rc = self._lib.gwg_stream_info(os.fsencode(path), ctypes.byref(kind), dims,
                                       ctypes.byref(complete), ctypes.byref(st))
        if rc != nat.GWG_OK:
            raise_for(st)
        self.t = int(dims[1])

    def run_grid_files(self, snps_path: str, out_path: str, rotated: bool = False,
                       mb: int = 0) -> dict:
        """run_grid over GWG1 files: SNP stream in, result stream out
        (gwg_run_grid_files; the output is finalized only on success)."""
        opts = nat.RunOptions()
        opts.mb, opts.layout, opts.double_buffer = int(mb), nat.GWG_LAYOUT_STREAM, 1
        cnt = nat.Counters()
        st = nat.Status()
        try:
            rc = self._lib.gwg_run_grid_files(self._h, os.fsencode(snps_path), int(rotated),
                                              os.fsencode(out_path), ctypes.byref(opts),
                                              ctypes.byref(cnt), ctypes.byref(st))
        finally:
            self._synced()
        if rc != nat.GWG_OK:
            raise_for(st)
        return cnt.as_dict()

    def counters(self) -> dict:
        c = nat.Counters()
        self._lib.gwg_get_counters(self._h, ctypes.byref(c))
        return c.as_dict()

    def reset_counters(self) -> None:
        self._lib.gwg_reset_counters(self._h)

    def synchronize(self) -> None:
        try:
            self._call(self._lib.gwg_synchronize)
        finally:
            self._synced()

    def wait_stream(self, stream) -> None:
        """Order the engine after work queued on a CUDA stream (a
        torch.cuda.Stream or a raw cudaStream_t)."""
        handle = getattr(stream, "cuda_stream", stream)
        self._call(self._lib.gwg_wait_stream, int(handle))

    def default_slab_snps(self, m: int) -> int:
        """The slab width run_grid uses for m SNP columns when mb = 0."""
        return int(self._lib.gwg_default_slab_snps(self._h, int(m)))

    @property
    def compute_stream(self) -> int:
        return int(self._lib.gwg_compute_stream(self._h) or 0)


class Group:
    """One process, several GPUs (gwg_group_*): one Engine per listed device
    (a device may repeat); shared operands go host -> the first device once
    and are broadcast device-to-device; run_grid shards m into contiguous
    balanced column ranges, one host thread and pinned pipeline per device,
    no other collective.  Results are bitwise those of a single Engine."""

    def __init__(self, n: int, p: int, devices):
        self._lib = nat.load()
        self.n, self.p, self.t = int(n), int(p), 0
        self.devices = [int(d) for d in devices]
        arr = (ctypes.c_int32 * len(self.devices))(*self.devices)
        st = nat.Status()
        self._h = self._lib.gwg_group_create(arr, len(self.devices), self.n, self.p,
                                             ctypes.byref(st))
        if not self._h:
            raise_for(st)
            raise DimensionError("device group creation failed")
        self.engines = [Engine(self.n, self.p, d, _handle=self._lib.gwg_group_engine(self._h, k))
                        for k, d in enumerate(self.devices)]

    def close(self) -> None:
        if getattr(self, "_h", None):
            for e in self.engines:
                e.close()
            self._lib.gwg_group_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, fn, *args) -> None:
        st = nat.Status()
        rc = fn(self._h, *args, ctypes.byref(st))
        if rc != nat.GWG_OK:
            raise_for(st)

    def shards(self, m: int) -> list[int]:
        bounds = (ctypes.c_int64 * (len(self.devices) + 1))()
        self._lib.gwg_group_shards(self._h, int(m), bounds)
        return list(bounds)

    def set_spectrum(self, basis, values) -> None:
        b = _Operand(basis, (self.n, self.n), "basis")
        v = _Operand(values, (self.n,), "values")
        self._call(self._lib.gwg_group_set_spectrum, b.ptr, v.ptr, b.where)

    def set_covariates(self, xl) -> None:
        if self.p == 1:
            self._call(self._lib.gwg_group_set_covariates, None, nat.GWG_HOST)
            return
        x = _Operand(xl, (self.n, self.p - 1), "xl")
        self._call(self._lib.gwg_group_set_covariates, x.ptr, x.where)

    def set_traits(self, traits, h2, sigma2, rotated: bool = False) -> None:
        t = int(np.shape(traits)[1]) if np.ndim(traits) == 2 else 1
        y = _Operand(traits if np.ndim(traits) == 2 else np.reshape(traits, (-1, 1)),
                     (self.n, t), "traits")
        h = _Operand(h2, (t,), "h2")
        s = _Operand(sigma2, (t,), "sigma2")
        if not (y.where == h.where == s.where):
            raise DimensionError("traits, h2 and sigma2 must live on the same side")
        self._call(self._lib.gwg_group_set_traits, t, y.ptr, h.ptr, s.ptr, y.where, int(rotated))
        self.t = t
        for e in self.engines:
            e.t = t
        if y.where == nat.GWG_DEVICE:  # the broadcast reads them asynchronously
            for e in self.engines:
                e.synchronize()

    def set_snp_coding(self, coding: str) -> None:
        code = {"real": nat.GWG_SNP_REAL, "genotypes": nat.GWG_SNP_GENOTYPES,
                "auto": nat.GWG_SNP_AUTO}.get(coding)
        if code is None:
            raise DimensionError(f"unknown SNP coding {coding!r}")
        self._call(self._lib.gwg_group_set_snp_coding, code)

    def set_option(self, name: str, value: int) -> None:
        if name not in nat.OPTIONS:
            raise DimensionError(f"unknown option {name!r}")
        self._call(self._lib.gwg_group_set_option, nat.OPTIONS[name], int(value))

    def run_grid(self, snps, out=None, layout: str = "numpy", mb: int = 0,
                 double_buffer: bool = True, checksum: bool = False, i0: int = 0,
                 sink=None, ring: int = 0, ldb: int = 0):
        """Engine.run_grid over every device of the group (m sharded); the
        sink, if any, is called from several threads (one per device)."""
        snps, fmt = _snp_array(snps, self.n)
        m = snps.shape[1]
        opts, out, out_ptr, keep, errors = _run_options(self.t, self.p, m, layout, mb,
                                                        double_buffer, checksum, i0, sink,
                                                        ring, ldb, fmt, out)
        cnt = nat.Counters()
        st = nat.Status()
        rc = self._lib.gwg_group_run_grid(self._h, m, snps.ctypes.data, out_ptr,
                                          ctypes.byref(opts), ctypes.byref(cnt), ctypes.byref(st))
        self.last_counters = cnt.as_dict()
        del keep
        if errors:
            raise errors[0]
        if rc != nat.GWG_OK:
            raise_for(st)
        return out

    def counters(self) -> dict:
        """Counters of the last run_grid (summed over devices; wall and stall
        of the slowest)."""
        return dict(getattr(self, "last_counters", {}))


def _dims_of(kinship, xl, snps, traits, h2, sigma2):
    """ProblemDims checks of bindings.cpp:100-113 + types.cpp:7-17."""
    kinship = np.asarray(kinship, dtype=np.float64)
    xl = np.asarray(xl, dtype=np.float64)
    snps = np.asarray(snps)
    if snps.dtype != np.int8:
        snps = snps.astype(np.float64, copy=False)
    traits = np.asarray(traits, dtype=np.float64)
    h2 = np.asarray(h2, dtype=np.float64).reshape(-1)
    sigma2 = np.asarray(sigma2, dtype=np.float64).reshape(-1)
    if xl.ndim == 1:
        xl = xl.reshape(-1, 1)
    n = kinship.shape[0]
    p = xl.shape[1] + 1
    m, t = snps.shape[1], traits.shape[1]
    if kinship.ndim != 2 or kinship.shape[1] != n or xl.shape[0] != n or snps.shape[0] != n \
            or traits.shape[0] != n:
        raise DimensionError("operand row counts disagree")
    if h2.shape[0] != t or sigma2.shape[0] != t:
        raise DimensionError("h2 and sigma2 must have one entry per trait")
    if n < 1:
        raise DimensionError(f"n must be >= 1, got {n}")
    if p > n:
        raise DimensionError(f"p ({p}) must not exceed n ({n}): each cell system is p x p "
                             "built from n samples")
    if m < 1:
        raise DimensionError(f"m must be >= 1, got {m}")
    if t < 1:
        raise DimensionError(f"t must be >= 1, got {t}")
    return kinship, xl, snps, traits, h2, sigma2, (n, p, m, t)


def device_working_set_bytes(n: int, p: int, t: int, mb: int, snp_coding: str = "real") -> int:
    """Resident HBM bytes of a run_grid with mb-column slabs (the device
    analogue of working_set_bytes, grid.cpp:279-297): spectrum, covariates,
    trait operands + contexts, two raw slabs, rotated slab(s), two result
    slabs; the FP64 path's factorised S_BR (E, F, G, S_BR) for t >= 256; for
    genotype coding also Z^T, the W build (V, W, int8 slices, and for t >= 256
    the factorised covariate panels diag(X_L'_c) E and Z diag(X_L'_c) E), the
    D panels, Z slices, the int8 slab and S_BR."""
    np_ = -(-n // 32) * 32
    kp = -(-n // 128) * 128
    r = 512                                                   # low-rank S_BR terms (max)
    fixed = (n * n + n) * 8 + 2 * n * max(p - 1, 1) * 8
    traits = (2 * n * t + 2 * t) * 8 + (-(-t // 8) * 8) * np_ * (p + 1) * 8 + t * (2 * p + p * p // 2) * 8
    per_snp = (2 * n + 2 * np_) * 8 + 2 * t * p * 8
    total = fixed + traits + mb * per_snp
    lowrank = r * np_ * 8 + (-(-t // 64) * 64) * r * 8       # E, F
    if t >= 256:                                              # FP64 path: G, S_BR of the slab
        total += lowrank + mb * (r + t) * 8
    if snp_coding in ("genotypes", "auto"):
        p8 = 1 << max(0, (p - 1).bit_length()) if p <= 8 else -(-p // 8) * 8
        kt = max(1, 32 // p8)
        wrows = -(-t // kt) * kt * p8
        total += np_ * n * 8 + 8 * n * kp + n * 8             # Z^T, Z slices + scales
        total += 2 * np_ * wrows * 8 + 8 * wrows * kp + wrows * 8  # V, W, W slices + scales
        total += -(-t // 64) * 64 * np_ * 8                   # D panels
        total += mb * (kp + t * 8)                            # int8 slab, S_BR
        if t < 256:
            total += lowrank + mb * r * 8                     # E, F, G
        elif p > 1:                                           # factorised covariate columns
            total += (np_ + n) * r * (p - 1) * 8              # (+ up to 16 split-K partials of U)
            total += 16 * n * r * (p - 1) * 8
    return total


def exp_sum_design(x_min: float, x_max: float, multiple: int = 64,
                   max_terms: int = 512) -> tuple[np.ndarray, np.ndarray]:
    """Nodes s and weights w of the positive exponential sum
    1/x ~= sum_r w[r] exp(-s[r] x) on [x_min, x_max] that factorises the GLS
    weights D for the genotype grid's S_BR term (csrc/expsum.cpp)."""
    lib = nat.load()
    r = ctypes.c_int32(0)
    rc = lib.gwg_exp_sum_design(float(x_min), float(x_max), int(multiple), int(max_terms),
                                None, None, ctypes.byref(r))
    if rc != 0:
        raise DimensionError(f"no exponential sum for [{x_min}, {x_max}] within {max_terms} terms")
    s = np.empty(r.value)
    w = np.empty(r.value)
    lib.gwg_exp_sum_design(float(x_min), float(x_max), int(multiple), int(max_terms),
                           s.ctypes.data, w.ctypes.data, ctypes.byref(r))
    return s, w


def solve_grid(kinship, xl, snps, traits, h2, sigma2, scheduler: str = "ct", workers: int = 1,
               nb: int = 0, mb: int = 0, tb: int = 0, mbb: int = 0, tbb: int = 0,
               double_buffer: bool = True, memory_budget: int | None = None,
               device: int = 0, device_eig: bool = False, snp_coding: str = "auto",
               devices=None, checksum: bool = False) -> dict:
    """Solve the whole m x t grid; returns {'b': (m, t, p), 'counters': dict}.

    Same signature and semantics as gwgrid.solve_grid (bindings.cpp:115-190,
    318-328).  ``scheduler``/``workers``/``nb``/``tb``/``mbb``/``tbb`` are the
    reference's CPU tiling knobs: they are validated with the reference's
    rules (grid.cpp:64-77) and have no effect on the result, which is bitwise
    independent of tiling here as well.  ``mb`` is the streamed SNP slab
    width.  ``memory_budget`` bounds the device working set.  ``device_eig``
    moves the one-off eigendecomposition to the GPU (cuSOLVER); by default it
    runs on the CPU like the reference.  ``snp_coding``: "auto" (default)
    picks, per slab, the exact int8 tensor-core path when every value is an
    integer genotype code and the FP64 path otherwise; "genotypes" requires
    codes, "real" always takes the FP64 path (see Engine.set_snp_coding);
    int8 ``snps`` travel as 1-byte codes.  ``devices`` (a list of GPU
    indices) shards m over a device Group; the result is bitwise the same.
    ``checksum`` adds the order-independent device checksum of b to the
    counters.
    """
    kinship, xl, snps, traits, h2, sigma2, (n, p, m, t) = _dims_of(
        kinship, xl, snps, traits, h2, sigma2)
    if scheduler not in ("ct", "it", "naive"):
        raise DimensionError("scheduler must be ct, it, or naive")
    for name, val, hi in (("nb", nb, m), ("mb", mb, m), ("tb", tb, t)):
        if val and not 1 <= val <= hi:
            raise DimensionError(f"tile parameter {name} out of range (got {val})")
    if mbb and not 1 <= mbb <= (mb or m):
        raise DimensionError(f"tile parameter mbb (must be in [1, mb]) out of range (got {mbb})")
    if tbb and not 1 <= tbb <= (tb or t):
        raise DimensionError(f"tile parameter tbb (must be in [1, tb]) out of range (got {tbb})")
    if memory_budget is not None:
        need1 = device_working_set_bytes(n, p, t, 1, snp_coding)
        if need1 > memory_budget:
            raise InfeasibleBudgetError(
                f"memory budget of {memory_budget} bytes cannot hold even a 1-column slab "
                f"(working set {need1} bytes)")
        if not mb:
            ws = [device_working_set_bytes(n, p, t, k, snp_coding) for k in (0, 1)]
            mb = max(1, min(m, (memory_budget - ws[0]) // (ws[1] - ws[0])))
        elif device_working_set_bytes(n, p, t, mb, snp_coding) > memory_budget:
            need = device_working_set_bytes(n, p, t, mb, snp_coding)
            raise InfeasibleBudgetError(
                f"working set of {need} bytes exceeds the memory budget of {memory_budget} bytes")
    b = np.empty((m, t, p), dtype=np.float64)
    t0 = time.perf_counter()
    if devices is not None and len(devices) > 0:
        if device_eig:
            raise DimensionError("device_eig is a single-device option")
        runner = Group(n, p, devices)
        basis, values = eigendecompose(kinship)
    else:
        runner = Engine(n, p, device)
        basis = values = None
    with runner as eng:
        if device_eig:
            eng.set_kinship(kinship)
        else:
            if basis is None:
                basis, values = eigendecompose(kinship)
            eng.set_spectrum(basis, values)
        eng.set_covariates(xl)
        preloop_s = time.perf_counter() - t0
        eng.set_snp_coding(snp_coding)
        eng.set_traits(traits, h2, sigma2)
        eng.run_grid(snps, b, mb=mb, double_buffer=double_buffer, checksum=checksum)
        c = eng.counters()
    stall = c["io_stall_ms"] * 1e-3
    wall = c["wall_ms"] * 1e-3
    counters = {
        "preloop_flops": int(c["preloop_flops"]),
        "loop_flops": int(c["loop_flops"]),
        "loop_transform_flops": 0,
        "context_builds": int(c["context_builds"]),
        "bytes_loaded": int(c["bytes_loaded"]),
        "bytes_stored": int(c["bytes_stored"]),
        "io_stall_seconds": stall,
        "loops_wall_seconds": wall,
        "preloop_wall_seconds": preloop_s,
        "stall_fraction": stall / wall if wall > 0 else 0.0,
        "grid_flops": int(c["grid_flops"]),
        "grid_kernel_seconds": c["grid_kernel_ms"] * 1e-3,
        "kernel_launches": int(c["kernel_launches"]),
    }
    if checksum:
        counters["checksum"] = int(c["checksum"])
        counters["checksum_cells"] = int(c["checksum_cells"])
    return {"b": b, "counters": counters}


def verify_grid(kinship, xl, snps, traits, h2, sigma2, b, device: int = 0,
                cell_errors: bool = False):
    """Max norm-wise relative error of b against the independent Cholesky
    route over every cell (gwgrid.verify_grid, bindings.cpp:192-222), computed
    on the device (gwg_verify_grid).  With ``cell_errors`` also returns the
    (m, t) array of per-cell errors."""
    kinship, xl, snps, traits, h2, sigma2, (n, p, m, t) = _dims_of(
        kinship, xl, snps, traits, h2, sigma2)
    snps = snps.astype(np.float64, copy=False)
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if b.shape != (m, t, p):
        raise DimensionError("b must have shape (m, t, p)")
    f = lambda a: np.asfortranarray(a)  # noqa: E731
    kinship, xl, snps, traits = f(kinship), f(xl), f(snps), f(traits)
    h2, sigma2 = np.ascontiguousarray(h2), np.ascontiguousarray(sigma2)
    out = ctypes.c_double(0.0)
    cells = np.empty((m, t), dtype=np.float64) if cell_errors else None
    st = nat.Status()
    rc = nat.load().gwg_verify_grid(int(device), n, p, m, t, kinship.ctypes.data,
                                    xl.ctypes.data if p > 1 else None, snps.ctypes.data,
                                    traits.ctypes.data, h2.ctypes.data, sigma2.ctypes.data,
                                    b.ctypes.data, cells.ctypes.data if cells is not None else None,
                                    ctypes.byref(out), ctypes.byref(st))
    if rc != nat.GWG_OK:
        raise_for(st)
    return (float(out.value), cells) if cell_errors else float(out.value)


def solve_cell(phi, xl, xr, y, h2: float, sigma2: float, device: int = 0) -> np.ndarray:
    """One fit via the eigendecomposition route (gwgrid.solve_cell,
    bindings.cpp:293-305), computed by the device engine."""
    phi = np.asarray(phi, dtype=np.float64)
    n = phi.shape[0]
    xl = np.asarray(xl, dtype=np.float64).reshape(n, -1)
    res = solve_grid(phi, xl, np.asarray(xr, dtype=np.float64).reshape(n, 1),
                     np.asarray(y, dtype=np.float64).reshape(n, 1), [h2], [sigma2],
                     device=device)
    return res["b"][0, 0].copy()
