"""BED1 batch files: the reference's bit-exact binary
batch format (/root/reference/pkg/src/batchedeig/core.py:312-395).

Layout: magic ``BED1``, then little-endian u32 version (= 1), batch, rows,
cols, then batch * rows * cols little-endian float64 values, matrices
concatenated, each row-major.  Round trips are bit-exact.  Accepts paths or
binary streams; torch tensors are written from the host copy.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .core import (
    BadMagic,
    BatchedMatrix,
    BatchedSymmetric,
    DimMismatch,
    TruncatedPayload,
)

__all__ = ["write_batch", "read_batch", "read_matrix"]

MAGIC = b"BED1"
VERSION = 1
_HDR = struct.Struct("<4I")  # version, batch, rows, cols


def _open(stream, mode):
    if isinstance(stream, (str, Path)):
        return open(stream, mode), True
    return stream, False


def _host_f64(data) -> np.ndarray:
    if hasattr(data, "detach"):  # torch tensor
        data = data.detach().cpu().numpy()
    return np.ascontiguousarray(data, dtype="<f8")


def write_batch(a, stream) -> None:
    """Write a BatchedSymmetric / BatchedMatrix (or a (batch, rows, cols) array)."""
    data = _host_f64(a.data if isinstance(a, (BatchedSymmetric, BatchedMatrix)) else a)
    if data.ndim != 3:
        raise DimMismatch(f"expected (batch, rows, cols), got {data.shape}")
    f, owned = _open(stream, "wb")
    try:
        b, rows, cols = data.shape
        f.write(MAGIC + _HDR.pack(VERSION, b, rows, cols) + data.tobytes())
    finally:
        if owned:
            f.close()


def _read(f) -> np.ndarray:
    if f.read(4) != MAGIC:
        raise BadMagic(f"stream does not start with {MAGIC!r}")
    head = f.read(_HDR.size)
    if len(head) < _HDR.size:
        raise TruncatedPayload("header truncated")
    version, b, rows, cols = _HDR.unpack(head)
    if version != VERSION:
        raise BadMagic(f"unsupported BED version {version}")
    if min(b, rows, cols) < 1:
        raise DimMismatch(f"invalid header counts batch={b} rows={rows} cols={cols}")
    want = 8 * b * rows * cols
    payload = f.read(want)
    if len(payload) < want:
        raise TruncatedPayload(f"payload holds {len(payload) // 8} reals, header announced {want // 8}")
    return np.frombuffer(payload, dtype="<f8").astype(np.float64).reshape(b, rows, cols)


def read_matrix(stream) -> BatchedMatrix:
    """Any BED1 batch (square or not)."""
    f, owned = _open(stream, "rb")
    try:
        return BatchedMatrix(_read(f))
    finally:
        if owned:
            f.close()


def read_batch(stream) -> BatchedSymmetric:
    """A square BED1 batch as symmetric input (symmetry is checked by the solve)."""
    f, owned = _open(stream, "rb")
    try:
        data = _read(f)
    finally:
        if owned:
            f.close()
    if data.shape[1] != data.shape[2]:
        raise DimMismatch(f"symmetric batch needs rows == cols, got {data.shape[1]}x{data.shape[2]}")
    return BatchedSymmetric(data)
