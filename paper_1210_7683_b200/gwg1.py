"""GWG1 binary streams (proj/include/gwgrid/stream.hpp:15-41), host side.

64-byte little-endian header — magic "GWG1", u16 version 1, u8 kind
(1 variant stream, 2 trait stream, 3 result grid, 4 operand matrix), u8
element type 0 (float64), u64 dims[3], u8 layout 0, u8 completeness
(0 = complete), zero padding — then a float64 payload: column-major for kinds
1/2/4 (the trait stream appends h2[t] and sigma2[t]); result cell (i, j) at
element (j*m + i)*p.  Writers create files incomplete and finalize them last;
readers reject incomplete, truncated or mistyped files (stream.cpp:219-257).
The engine reads and writes the same format natively (gwg_run_grid_files).
"""
from __future__ import annotations

import os
import struct

import numpy as np

from .errors import IoError

KIND_SNP, KIND_TRAIT, KIND_RESULT, KIND_OPERAND = 1, 2, 3, 4
HEADER = 64
_NAMES = {1: "variant stream", 2: "trait stream", 3: "result grid", 4: "operand matrix"}


def encode_header(kind: int, dims: tuple, complete: bool = True) -> bytes:
    d = tuple(dims) + (0,) * (3 - len(dims))
    head = b"GWG1" + struct.pack("<HBB3QBB", 1, kind, 0, *d, 0, 0 if complete else 1)
    return head + bytes(HEADER - len(head))


def payload_bytes(kind: int, dims: tuple) -> int:
    d0, d1, d2 = (tuple(dims) + (0, 0, 0))[:3]
    if kind in (KIND_SNP, KIND_OPERAND):
        return d0 * d1 * 8
    if kind == KIND_TRAIT:
        return d1 * (d0 + 2) * 8
    return d0 * d1 * d2 * 8


def read_header(path: str, expected_kind: int | None = None) -> dict:
    """Parse and validate a header like InputStream::open."""
    size = os.path.getsize(path)
    if size < HEADER:
        raise IoError(f"{path} is shorter than the header ({size} of {HEADER} bytes)")
    with open(path, "rb") as f:
        b = f.read(HEADER)
    if b[:4] != b"GWG1":
        raise IoError(f"bad magic in {path} (not a GWG1 stream)")
    version, kind, etype = struct.unpack_from("<HBB", b, 4)
    dims = struct.unpack_from("<3Q", b, 8)
    layout, incomplete = b[32], b[33]
    if version != 1:
        raise IoError(f"unsupported stream version {version} in {path} (expected 1)")
    if kind not in _NAMES:
        raise IoError(f"unknown stream kind {kind} in {path}")
    if etype != 0:
        raise IoError(f"unsupported element type {etype} in {path}")
    if layout != 0:
        raise IoError(f"unsupported layout {layout} in {path}")
    if expected_kind is not None and kind != expected_kind:
        raise IoError(f"{path} holds a {_NAMES[kind]}, expected a {_NAMES[expected_kind]}")
    if incomplete:
        raise IoError(f"{path} was never finalized by its writer")
    want = HEADER + payload_bytes(kind, dims)
    if size != want:
        raise IoError(f"{path} has {size} bytes, header promises {want}")
    return {"kind": kind, "dims": dims}


def write_columns_stream(path: str, kind: int, cols: np.ndarray, extra: tuple = ()) -> None:
    a = np.asfortranarray(np.asarray(cols, dtype=np.float64))
    with open(path, "wb") as f:
        f.write(encode_header(kind, (a.shape[0], a.shape[1], 0), complete=False))
        f.write(a.tobytes(order="F"))
        for e in extra:
            f.write(np.ascontiguousarray(e, dtype=np.float64).tobytes())
        f.flush()
        f.seek(33)
        f.write(b"\x00")  # finalize


def write_snp_stream(path: str, snps: np.ndarray) -> None:
    """Kind 1: n x m variant columns."""
    write_columns_stream(path, KIND_SNP, snps)


def write_trait_stream(path: str, traits: np.ndarray, h2, sigma2) -> None:
    """Kind 2: n x t trait columns, then h2[t] and sigma2[t]."""
    t = np.shape(traits)[1]
    h2 = np.asarray(h2, dtype=np.float64).reshape(t)
    sigma2 = np.asarray(sigma2, dtype=np.float64).reshape(t)
    write_columns_stream(path, KIND_TRAIT, traits, (h2, sigma2))


def read_columns(path: str, expected_kind: int = KIND_SNP) -> np.ndarray:
    h = read_header(path, expected_kind)
    n, m = h["dims"][0], h["dims"][1]
    return np.fromfile(path, dtype="<f8", count=n * m, offset=HEADER).reshape((n, m), order="F")


def read_result(path: str, layout: str = "numpy") -> np.ndarray:
    """Kind 3 result grid as (m, t, p) ("numpy") or its native (t, m, p)."""
    h = read_header(path, KIND_RESULT)
    m, t, p = h["dims"]
    raw = np.memmap(path, dtype="<f8", mode="r", offset=HEADER, shape=(t, m, p))
    return np.ascontiguousarray(raw.transpose(1, 0, 2)) if layout == "numpy" else np.array(raw)
