"""MDPMAT01 binary matrices straight into HBM (reference fileio.py:1-105).

Layout (little-endian): magic "MDPMAT01" | kind u8 (0 dense, 1 CSR) | rows u64
| cols u64 | nnz u64 | payload (dense: rows*cols f64 row-major; CSR: row_ptr
(rows+1) u64, col_idx nnz u64, values nnz f64).  The header arithmetic is
checked against the file length before the payload is touched, and errors
carry byte offsets (FileFormatError, fileio.py:35-40).  The payload is
memory-mapped and uploaded once; u64 column indices are narrowed to the
device's int32 layout after a range check on the GPU (CsrMatrix check).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from .sparse import CsrMatrix

MAGIC = b"MDPMAT01"
KIND_DENSE = 0
KIND_CSR = 1
HEADER_LEN = 33
_HEADER = struct.Struct("<8sBQQQ")

__all__ = ["FileFormatError", "read_matrix", "write_matrix"]


class FileFormatError(ValueError):
    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (at byte offset {offset})")
        self.offset = offset


def write_matrix(path, matrix) -> None:
    path = Path(path)
    if isinstance(matrix, CsrMatrix):
        rp, ci, va = matrix.numpy()
        with open(path, "wb") as fh:
            fh.write(_HEADER.pack(MAGIC, KIND_CSR, matrix.rows, matrix.cols, matrix.nnz))
            fh.write(rp.astype("<u8").tobytes())
            fh.write(ci.astype("<u8").tobytes())
            fh.write(va.astype("<f8").tobytes())
        return
    dense = matrix.detach().cpu().numpy() if isinstance(matrix, torch.Tensor) else \
        np.asarray(matrix, dtype=np.float64)
    if dense.ndim != 2:
        raise ValueError(f"dense matrices must be 2-D, got shape {dense.shape}")
    rows, cols = dense.shape
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, KIND_DENSE, rows, cols, rows * cols))
        fh.write(np.ascontiguousarray(dense, dtype="<f8").tobytes())


def read_matrix(path):
    """ndarray (dense) or device CsrMatrix."""
    path = Path(path)
    size = path.stat().st_size
    if size < HEADER_LEN:
        raise FileFormatError(f"file is {size} bytes, shorter than the header", size)
    with open(path, "rb") as fh:
        magic, kind, rows, cols, nnz = _HEADER.unpack(fh.read(HEADER_LEN))
    if magic != MAGIC:
        raise FileFormatError(f"bad magic {magic!r}, expected {MAGIC!r}", 0)
    if kind not in (KIND_DENSE, KIND_CSR):
        raise FileFormatError(f"unknown matrix kind {kind}", 8)
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    if kind == KIND_DENSE:
        if nnz != rows * cols:
            raise FileFormatError(f"dense header declares nnz={nnz}, expected rows*cols={rows * cols}", 25)
        expected = HEADER_LEN + 8 * rows * cols
        if size != expected:
            raise FileFormatError(f"file length {size} does not match header arithmetic {expected}",
                                  min(size, expected))
        return np.frombuffer(mm, dtype="<f8", count=rows * cols, offset=HEADER_LEN).astype(
            np.float64).reshape(rows, cols)
    expected = HEADER_LEN + 8 * (rows + 1) + 16 * nnz
    if size != expected:
        raise FileFormatError(f"file length {size} does not match header arithmetic {expected}",
                              min(size, expected))
    off = HEADER_LEN
    row_ptr = np.frombuffer(mm, dtype="<u8", count=rows + 1, offset=off).astype(np.int64)
    off += 8 * (rows + 1)
    if row_ptr[-1] != nnz:
        raise FileFormatError(f"row_ptr ends at {row_ptr[-1]} but the header declares nnz={nnz}",
                              off - 8)
    col_idx = np.frombuffer(mm, dtype="<u8", count=nnz, offset=off)
    off += 8 * nnz
    values = np.frombuffer(mm, dtype="<f8", count=nnz, offset=off)
    big = col_idx.size and int(col_idx.max()) >= 2 ** 31
    cols_i = np.where(col_idx >= 2 ** 31, np.uint64(2 ** 31 - 1), col_idx).astype(np.int64) if big \
        else col_idx.astype(np.int64)
    try:
        return CsrMatrix(rows, cols, row_ptr, cols_i, values.astype(np.float64))
    except ValueError as exc:
        raise FileFormatError(f"payload is not a valid CSR matrix: {exc}", HEADER_LEN) from exc
