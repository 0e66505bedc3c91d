"""Binary CSR container (.csrb) shared with tools/condkit_b200_cli:

    b"CKCSR001" | int64 nrows, ncols, nnz | int64 row_offsets[nrows + 1] |
    int32 col_indices[nnz] | float64 values[nnz]

Loading is a few sequential reads (no text parsing), so operators of
hundreds of millions of entries reach the device in seconds.
"""
from __future__ import annotations

import numpy as np

from .sparse import SparseMatrix

MAGIC = b"CKCSR001"


def write_csrb(a: SparseMatrix, path: str) -> None:
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(np.array([a.nrows, a.ncols, a.nnz], np.int64).tobytes())
        f.write(np.ascontiguousarray(a.row_offsets, np.int64).tobytes())
        f.write(np.ascontiguousarray(a.col_indices, np.int32).tobytes())
        f.write(np.ascontiguousarray(a.values, np.float64).tobytes())


def read_csrb(path: str, validate: bool = True) -> SparseMatrix:
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError(f"not a .csrb file: {path}")
        nr, nc, nnz = (int(v) for v in np.fromfile(f, np.int64, 3))
        rp = np.fromfile(f, np.int64, nr + 1)
        ci = np.fromfile(f, np.int32, nnz)
        va = np.fromfile(f, np.float64, nnz)
    if rp.size != nr + 1 or ci.size != nnz or va.size != nnz:
        raise ValueError(f"truncated .csrb file: {path}")
    return SparseMatrix(nr, nc, rp, ci, va, validate=validate)
