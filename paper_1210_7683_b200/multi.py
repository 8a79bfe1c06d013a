"""Multi-GPU plumbing for one process per GPU (torchrun / torch.distributed).

SURVEY §8e: every (i, j) cell is independent, so the SNP axis m shards into
contiguous column ranges, one per rank.  The shared operands — the kinship
eigensystem Z, lambda, the covariates X_L, the traits Y, h2 and sigma2 — are
produced once on rank 0 (the CPU eigendecomposition is the one-off preloop)
and broadcast once (NCCL over NVLink / NVSwitch on a GPU node, gloo on CPU);
each rank then generates or loads only its own SNP shard, solves it and owns
disjoint result rows.  There is no data-path collective: the only traffic
after the broadcast is one gather of 8-byte checksums (and of timings, in
bench.py).  The reference has no distributed layer; this is the
device-count analogue of run_grid's IT scheduler, where each worker owns
slabs k = w (mod workers) (proj/src/grid.cpp:559-639).

The single-process alternative (one host thread per GPU, peer copies instead
of NCCL) is ``engine.Group``; both split m exactly like ``shard_bounds``.

``solve_sharded`` takes the per-rank solve as a callable, so the same driver
runs the device engine (``engine_compute``) on GPUs and the CPU oracle in the
gloo tests.
"""
from __future__ import annotations

import os
from typing import Callable

import numpy as np

SHARED_KEYS = ("basis", "values", "xl", "y", "h2", "sigma2")


def shard_bounds(m: int, world: int) -> list[int]:
    """Contiguous balanced shards: rank k owns SNP columns
    [bounds[k], bounds[k+1]) (the formula of gwg_group_shards)."""
    if world < 1 or m < 0:
        raise ValueError("need world >= 1 and m >= 0")
    return [k * m // world for k in range(world + 1)]


def rank_range(m: int, world: int, rank: int) -> tuple[int, int]:
    b = shard_bounds(m, world)
    return b[rank], b[rank + 1]


def dist_env() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shared_shapes(n: int, p: int, t: int) -> dict:
    """Shapes of the shared operands, each stored as a contiguous tensor
    (matrices transposed: the engine reads them column-major)."""
    return {"basis": (n, n), "values": (n,), "xl": (max(p - 1, 0), n), "y": (t, n),
            "h2": (t,), "sigma2": (t,)}


def broadcast_shared(shared: dict | None, n: int, p: int, t: int, device=None,
                     src: int = 0) -> dict:
    """Rank ``src`` passes ``shared`` (numpy: basis (n, n) and xl (n, p-1) and
    y (n, t) column-major as (rows, cols), values/h2/sigma2 vectors); every
    rank returns torch tensors on ``device`` holding the same values, in the
    engine's column-major convention (matrices as transposed views).  One
    broadcast per operand, nothing else."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank() if dist.is_initialized() else 0
    shapes = shared_shapes(n, p, t)
    out = {}
    for key in SHARED_KEYS:
        if rank == src:
            a = np.asarray(shared[key], dtype=np.float64)
            if a.ndim == 2:
                a = np.ascontiguousarray(a.T)  # (cols, rows): contiguous column-major
            buf = torch.from_numpy(a).to(device) if device is not None else torch.from_numpy(a)
        else:
            buf = torch.empty(shapes[key], dtype=torch.float64, device=device)
        if dist.is_initialized():  # (a no-op at world size 1, kept to exercise the call)
            dist.broadcast(buf, src=src)
        out[key] = buf.t() if buf.dim() == 2 else buf
    return out


def gather_checksums(local: int) -> int:
    """Wrapping uint64 sum of every rank's checksum (one 8-byte all-gather)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return int(local) & 0xFFFFFFFFFFFFFFFF
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else None
    mine = torch.tensor([np.uint64(local).view(np.int64)], dtype=torch.int64, device=dev)
    parts = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, mine)
    total = 0
    for x in parts:
        total = (total + int(np.int64(x.item()).view(np.uint64))) & 0xFFFFFFFFFFFFFFFF
    return total


def solve_sharded(n: int, p: int, m: int, t: int, make_shared: Callable[[], dict],
                  load_shard: Callable[[int, int], np.ndarray],
                  compute: Callable[[dict, np.ndarray, int], tuple[np.ndarray, int]],
                  device=None) -> dict:
    """The sharded run: rank 0 builds the shared operands (make_shared), they
    are broadcast once, each rank loads its shard [i0, i1) (load_shard) and
    solves it (compute(shared, x_shard, i0) -> (b_local, checksum)).  Returns
    {"i0", "i1", "b": this rank's (i1 - i0, t, p) rows, "checksum": the
    whole grid's checksum}."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    shared = broadcast_shared(make_shared() if rank == 0 else None, n, p, t, device=device)
    i0, i1 = rank_range(m, world, rank)
    b, local = compute(shared, load_shard(i0, i1), i0)
    return {"i0": i0, "i1": i1, "b": b, "checksum": gather_checksums(local)}


def engine_compute(device: int, snp_coding: str = "auto", **run_kw):
    """compute() for solve_sharded on a GPU rank: one Engine on ``device``,
    the shared operands from HBM, the shard streamed by run_grid with global
    SNP indices and the device checksum."""
    from .engine import Engine

    def compute(shared: dict, x: np.ndarray, i0: int):
        n = shared["basis"].shape[0]
        p = shared["xl"].shape[1] + 1
        with Engine(n, p, device) as eng:
            eng.set_spectrum(shared["basis"], shared["values"])
            eng.set_covariates(shared["xl"])
            eng.set_snp_coding(snp_coding)
            eng.set_traits(shared["y"], shared["h2"], shared["sigma2"])
            b = eng.run_grid(x, checksum=True, i0=i0, **run_kw)
            return b, int(eng.counters()["checksum"])

    return compute
