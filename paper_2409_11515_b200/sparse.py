"""CSR container and device operator products.

Mirrors ``condkit::SparseMatrix`` (sparse.hpp:47-152): host-side CSR with the
same invariants, ``from_triplets`` (duplicates summed), ``identity`` and
``coeff``. ``matvec`` / ``transpose_matvec`` (sparse.hpp:212-242) run on the
B200 through the C-ABI and are bit-identical to the reference (stored-order
row sums; increasing-row accumulation for the transpose).

Storage: int64 row offsets, int32 column indices, float64 values (12 B per
nonzero on the device, versus 16 B for the reference's size_t indices).
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from .errors import DimensionMismatch, InvalidArgument, Unsupported, ZeroColumn, ZeroRow


class SparseMatrix:
    __slots__ = ("_nrows", "_ncols", "_rp", "_ci", "_va", "_dev", "__weakref__")

    def __init__(self, nrows: int, ncols: int, row_offsets, col_indices, values,
                 validate: bool = True):
        self._nrows, self._ncols = int(nrows), int(ncols)
        self._rp = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.asarray(col_indices)
        if ci.size and (ci.max(initial=0) >= 2**31 or ci.min(initial=0) < 0):
            raise DimensionMismatch("column index out of range")
        self._ci = np.ascontiguousarray(ci, dtype=np.int32)
        self._va = np.ascontiguousarray(values, dtype=np.float64)
        self._dev = None
        if validate:
            self._validate()

    # SparseMatrix::validate, sparse.hpp:129-145
    def _validate(self) -> None:
        rp, ci, va, n = self._rp, self._ci, self._va, self._nrows
        if (rp.size != n + 1 or rp[0] != 0 or rp[-1] != va.size or ci.size != va.size):
            raise DimensionMismatch("inconsistent CSR arrays")
        if n and np.any(np.diff(rp) < 0):
            raise DimensionMismatch("row offsets decrease")
        if ci.size:
            if ci.min() < 0 or ci.max() >= self._ncols:
                raise DimensionMismatch("column index out of range")
            d = np.diff(ci.astype(np.int64))
            starts = np.zeros(ci.size, dtype=bool)
            starts[rp[:-1][rp[:-1] < ci.size]] = True
            if np.any((d <= 0) & ~starts[1:]):
                raise DimensionMismatch("column indices not strictly increasing in a row")
            if not np.all(np.isfinite(va)):
                raise DimensionMismatch("non-finite entry")

    # sparse.hpp:67-96 (duplicates summed in input order)
    @staticmethod
    def from_triplets(nrows: int, ncols: int, entries) -> "SparseMatrix":
        t = list(entries)
        if not t:
            return SparseMatrix(nrows, ncols, np.zeros(nrows + 1, np.int64), [], [])
        r = np.array([e[0] for e in t], dtype=np.int64)
        c = np.array([e[1] for e in t], dtype=np.int64)
        v = np.array([e[2] for e in t], dtype=np.float64)
        return SparseMatrix.from_coo(nrows, ncols, r, c, v)

    @staticmethod
    def from_coo(nrows: int, ncols: int, r, c, v) -> "SparseMatrix":
        r = np.asarray(r, np.int64)
        c = np.asarray(c, np.int64)
        v = np.asarray(v, np.float64)
        if r.size and (r.min() < 0 or r.max() >= nrows or c.min() < 0 or c.max() >= ncols):
            raise DimensionMismatch(f"triplet index outside {nrows}x{ncols}")
        order = np.lexsort((c, r))  # stable: equal keys keep input order
        r, c, v = r[order], c[order], v[order]
        if r.size:
            new = np.ones(r.size, dtype=bool)
            new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            idx = np.flatnonzero(new)
            vs = np.array([v[a:b].sum() if b - a > 1 else v[a]
                           for a, b in zip(idx, list(idx[1:]) + [r.size])]) \
                if not np.all(new) else v
            r, c, v = r[idx], c[idx], vs
        rp = np.zeros(nrows + 1, np.int64)
        np.add.at(rp, r + 1, 1)
        rp = np.cumsum(rp)
        return SparseMatrix(nrows, ncols, rp, c, v)

    @staticmethod
    def identity(n: int) -> "SparseMatrix":
        return SparseMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n), np.ones(n))

    @property
    def nrows(self) -> int:
        return self._nrows

    @property
    def ncols(self) -> int:
        return self._ncols

    @property
    def nnz(self) -> int:
        return int(self._va.size)

    @property
    def row_offsets(self) -> np.ndarray:
        return self._rp

    @property
    def col_indices(self) -> np.ndarray:
        return self._ci

    @property
    def values(self) -> np.ndarray:
        return self._va

    def coeff(self, i: int, j: int) -> float:
        a, b = self._rp[i], self._rp[i + 1]
        k = a + np.searchsorted(self._ci[a:b], j)
        return float(self._va[k]) if k < b and self._ci[k] == j else 0.0

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self._nrows, self._ncols))
        rows = np.repeat(np.arange(self._nrows), np.diff(self._rp))
        np.add.at(d, (rows, self._ci), self._va)
        return d

    # ----------------------------------------------------------- device side
    def device(self) -> "DeviceMatrix":
        """The B200-resident operator (uploaded once, cached on this object)."""
        if self._dev is None:
            self._dev = DeviceMatrix(self)
        return self._dev

    def release_device(self) -> None:
        if self._dev is not None:
            self._dev.free()
            self._dev = None


class DeviceMatrix:
    """Handle of ``ck_matrix_upload``: A and A^T as sliced-ELL in HBM."""

    def __init__(self, a: SparseMatrix):
        lib = _lib.load()
        _lib.ensure_device()
        if a.nnz >= 2**32:
            raise Unsupported("nnz >= 2^32")
        h = C.c_void_p()
        _lib.check(lib.ck_matrix_upload(a.nrows, a.ncols, _lib.i64ptr(a.row_offsets),
                                        _lib.i32ptr(a.col_indices), _lib.dptr(a.values),
                                        C.byref(h)), "ck_matrix_upload")
        self.handle = h
        self.nrows, self.ncols, self.nnz = a.nrows, a.ncols, a.nnz
        self._fin = weakref.finalize(self, lib.ck_matrix_free, h)

    def free(self) -> None:
        self._fin()

    def info(self) -> dict:
        inf = _lib.MatrixInfo()
        _lib.check(_lib.load().ck_matrix_get_info(self.handle, C.byref(inf)), "ck_matrix_get_info")
        return {k: getattr(inf, k) for k, _ in _lib.MatrixInfo._fields_}

    def matvec(self, x) -> np.ndarray:
        x = _lib.as_f64(x, self.ncols, "matvec: vector")
        y = np.empty(self.nrows)
        _lib.check(_lib.load().ck_spmv(self.handle, _lib.dptr(x), _lib.dptr(y)), "ck_spmv")
        return y

    def transpose_matvec(self, x) -> np.ndarray:
        x = _lib.as_f64(x, self.nrows, "transpose_matvec: vector")
        y = np.empty(self.ncols)
        _lib.check(_lib.load().ck_spmv_t(self.handle, _lib.dptr(x), _lib.dptr(y)), "ck_spmv_t")
        return y

    def residual_norms(self, x, b):
        x = _lib.as_f64(x, self.ncols, "solution")
        b = _lib.as_f64(b, self.nrows, "rhs")
        rn, xn, bn = C.c_double(), C.c_double(), C.c_double()
        _lib.check(_lib.load().ck_residual_norms(self.handle, _lib.dptr(x), _lib.dptr(b),
                                                 C.byref(rn), C.byref(xn), C.byref(bn)),
                   "ck_residual_norms")
        return rn.value, xn.value, bn.value


def matvec(a: SparseMatrix, x) -> np.ndarray:
    """y = A x on the device (sparse.hpp:212-226)."""
    if np.asarray(x).size != a.ncols:
        raise DimensionMismatch(f"matvec: vector length {np.asarray(x).size} != ncols {a.ncols}")
    return a.device().matvec(x)


def transpose_matvec(a: SparseMatrix, x) -> np.ndarray:
    """y = A^T x on the device (sparse.hpp:230-242)."""
    if np.asarray(x).size != a.nrows:
        raise DimensionMismatch(
            f"transpose_matvec: vector length {np.asarray(x).size} != nrows {a.nrows}")
    return a.device().transpose_matvec(x)


# ------------------------------------------------------------------ scaling
class ScalingDiagonal:
    """Positive finite diagonal scaling factors (sparse.hpp:154-171)."""

    def __init__(self, factors):
        f = np.ascontiguousarray(factors, np.float64)
        bad = np.flatnonzero(~((f > 0.0) & np.isfinite(f)))
        if bad.size:
            raise InvalidArgument(f"scaling factor {int(bad[0])} is not positive and finite")
        self._f = f

    def __len__(self) -> int:
        return self._f.size

    def size(self) -> int:
        return self._f.size

    def __getitem__(self, i):
        return self._f[i]

    @property
    def factors(self) -> np.ndarray:
        return self._f


def column_norms(a: SparseMatrix) -> np.ndarray:
    """Euclidean norm of every column on the device (sparse.hpp:244-268), bit-identical."""
    out = np.empty(a.ncols)
    _lib.check(_lib.load().ck_column_norms(a.device().handle, _lib.dptr(out)), "column_norms")
    return out


def row_norms(a: SparseMatrix) -> np.ndarray:
    """two_norm of every row on the device (the row_scale factors)."""
    out = np.empty(a.nrows)
    _lib.check(_lib.load().ck_row_norms(a.device().handle, _lib.dptr(out)), "row_norms")
    return out


def column_scale(a: SparseMatrix):
    """(A D^-1, D) with D the column norms (sparse.hpp:270-284); ZeroColumn on the
    first zero-norm column."""
    vals = np.empty(a.nnz)
    norms = np.empty(a.ncols)
    zi = C.c_int64(-1)
    st = _lib.load().ck_column_scale(a.device().handle, _lib.i32ptr(a.col_indices),
                                     _lib.dptr(a.values), _lib.dptr(vals), _lib.dptr(norms),
                                     C.byref(zi))
    if st == ZeroColumn.status:
        raise ZeroColumn(_lib.load().ck_last_error().decode(), column=zi.value)
    _lib.check(st, "column_scale")
    scaled = SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, vals, validate=False)
    return scaled, ScalingDiagonal(norms)


def row_scale(a: SparseMatrix, b):
    """(D_r^-1 A, D_r^-1 b) with D_r the row norms (sparse.hpp:295-311); ZeroRow on
    the first zero-norm row."""
    b = np.ascontiguousarray(b, np.float64)
    if b.size != a.nrows:
        raise DimensionMismatch("row_scale: rhs length != nrows")
    vals = np.empty(a.nnz)
    bs = np.empty(a.nrows)
    norms = np.empty(a.nrows)
    zi = C.c_int64(-1)
    st = _lib.load().ck_row_scale(a.device().handle, _lib.i64ptr(a.row_offsets),
                                  _lib.dptr(a.values), _lib.dptr(vals), _lib.dptr(b),
                                  _lib.dptr(bs), _lib.dptr(norms), C.byref(zi))
    if st == ZeroRow.status:
        raise ZeroRow(_lib.load().ck_last_error().decode(), row=zi.value)
    _lib.check(st, "row_scale")
    return SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, vals, validate=False), bs


def unscale_solution(y, d: ScalingDiagonal) -> np.ndarray:
    """x = D^-1 y componentwise (sparse.hpp:286-293)."""
    y = np.ascontiguousarray(y, np.float64)
    f = d.factors if isinstance(d, ScalingDiagonal) else np.ascontiguousarray(d, np.float64)
    if y.size != f.size:
        raise DimensionMismatch("unscale_solution: length mismatch")
    x = np.empty(y.size)
    _lib.check(_lib.load().ck_unscale_solution(y.size, _lib.dptr(y), _lib.dptr(f), _lib.dptr(x)),
               "unscale_solution")
    return x
