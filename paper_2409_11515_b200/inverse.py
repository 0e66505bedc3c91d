"""||A^-1||_2 and kappa_2 on the device: LU factors, InverseOracle, cond2.

Mirror of the reference's lu.hpp / condest.hpp inverse half:
  LUFactors (lu.hpp:42-47), lu_factorize (:55-177), lu_solve (:180-202),
  lu_transpose_solve (:207-227), InverseOracle (condest.hpp:138-152),
  inv_norm2 (:320-322), Cond2Result / cond2 (:324-365).

The factors live on the B200 as a LAPACK-layout band LU with row partial
pivoting (csrc/ck_lu.cu); every solve and every Projected-Adam iteration on
A^-1 runs there (csrc/ck_inverse.cu).
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .condest import (AdamConfig, ExplicitOracle, GradientOracle, NormEstimate, Session,
                      estimate_norm)
from .errors import (DimensionMismatch, InvalidArgument, NumericallySingular,
                     StructurallySingular)
from .sparse import SparseMatrix


class LUFactors:
    """Device LU of a square SparseMatrix (P A = L U, band storage)."""

    def __init__(self, handle, n: int):
        self.handle = handle
        self._fin = weakref.finalize(self, _lib.load().ck_lu_free, handle)
        n_, kl, ku, pm, nb = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double(), C.c_int64()
        _lib.check(_lib.load().ck_lu_get_info(handle, C.byref(n_), C.byref(kl), C.byref(ku),
                                              C.byref(pm), C.byref(nb)), "ck_lu_get_info")
        self.n, self.kl, self.ku = n_.value, kl.value, ku.value
        self.pivot_min = pm.value
        self.device_bytes = nb.value
        self._csr = None

    def solve(self, b) -> np.ndarray:
        b = _lib.as_f64(b, self.n, "lu_solve: rhs")
        x = np.empty(self.n)
        _lib.check(_lib.load().ck_lu_solve(self.handle, _lib.dptr(b), _lib.dptr(x)), "lu_solve")
        return x

    def transpose_solve(self, b) -> np.ndarray:
        b = _lib.as_f64(b, self.n, "lu_transpose_solve: rhs")
        x = np.empty(self.n)
        _lib.check(_lib.load().ck_lu_transpose_solve(self.handle, _lib.dptr(b), _lib.dptr(x)),
                   "lu_transpose_solve")
        return x

    def dense_info(self):
        """(available, growth) of the dense-block sweeps the InverseOracle loop uses on
        narrow bands (ck_lu_dense_info): growth = max over 32-row blocks of
        || |Hinv| |H| ||_inf of the head triangles."""
        ok, g = C.c_int32(), C.c_double()
        _lib.check(_lib.load().ck_lu_dense_info(self.handle, C.byref(ok), C.byref(g)), "ck_lu_dense_info")
        return bool(ok.value), g.value

    def dense_solve(self, b, transpose: bool = False) -> np.ndarray:
        """lu_solve / lu_transpose_solve through the dense-block sweeps (parity tests)."""
        b = _lib.as_f64(b, self.n, "lu_dense_solve: rhs")
        x = np.empty(self.n)
        _lib.check(_lib.load().ck_lu_dense_solve(self.handle, 1 if transpose else 0, _lib.dptr(b),
                                                 _lib.dptr(x)), "lu_dense_solve")
        return x

    def export_csr(self):
        """(L, U, row_perm) in the reference's LUFactors shape (lu.hpp:42-47): L strictly
        lower in pivot coordinates (unit diagonal implicit), U upper with the diagonal
        first in each row, both CSR SparseMatrix; row_perm[k] = original row pivoted at
        step k. Assembled on the device (ck_lu_export_csr)."""
        if self._csr is None:
            lib = _lib.load()
            nl, nu = C.c_int64(), C.c_int64()
            _lib.check(lib.ck_lu_csr_info(self.handle, C.byref(nl), C.byref(nu)), "ck_lu_csr_info")
            n = self.n
            lrp, urp = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64)
            lci, uci = np.empty(max(nl.value, 1), np.int32), np.empty(max(nu.value, 1), np.int32)
            lva, uva = np.empty(max(nl.value, 1)), np.empty(max(nu.value, 1))
            perm = np.empty(n, np.int64)
            _lib.check(lib.ck_lu_export_csr(self.handle, _lib.i64ptr(lrp), _lib.i32ptr(lci),
                                            _lib.dptr(lva), _lib.i64ptr(urp), _lib.i32ptr(uci),
                                            _lib.dptr(uva), _lib.i64ptr(perm)), "ck_lu_export_csr")
            l = SparseMatrix(n, n, lrp, lci[: nl.value], lva[: nl.value], validate=False)
            u = SparseMatrix(n, n, urp, uci[: nu.value], uva[: nu.value], validate=False)
            self._csr = (l, u, perm)
        return self._csr

    @property
    def l(self) -> SparseMatrix:
        return self.export_csr()[0]

    @property
    def u(self) -> SparseMatrix:
        return self.export_csr()[1]

    @property
    def row_perm(self) -> np.ndarray:
        return self.export_csr()[2]

    def export_band(self):
        """(ab, ipiv) in LAPACK band layout: ab[kv + i - j, j] = factor(i, j)."""
        ldab = 2 * self.kl + self.ku + 1
        ab = np.empty(ldab * self.n)
        ipiv = np.empty(self.n, np.int32)
        _lib.check(_lib.load().ck_lu_export(self.handle, _lib.dptr(ab), _lib.i32ptr(ipiv)),
                   "ck_lu_export")
        return ab.reshape(self.n, ldab).T.copy(), ipiv


def lu_factorize(a: SparseMatrix, pivot_tol: float = 1e-12) -> LUFactors:
    """lu.hpp:55-177 on the device; raises Structurally/NumericallySingular."""
    if a.nrows != a.ncols:
        raise DimensionMismatch("lu_factorize: matrix must be square")
    h = C.c_void_p()
    col, piv = C.c_int64(-1), C.c_double(0.0)
    st = _lib.load().ck_lu_factorize(a.device().handle, pivot_tol, C.byref(h), C.byref(col),
                                     C.byref(piv))
    if st == StructurallySingular.status:
        raise StructurallySingular(_lib.load().ck_last_error().decode(), column=col.value)
    if st == NumericallySingular.status:
        raise NumericallySingular(_lib.load().ck_last_error().decode(), column=col.value,
                                  pivot=piv.value)
    _lib.check(st, "lu_factorize")
    return LUFactors(h, a.nrows)


def lu_solve(f: LUFactors, b) -> np.ndarray:
    return f.solve(b)


def lu_transpose_solve(f: LUFactors, b) -> np.ndarray:
    return f.transpose_solve(b)


class InverseOracle(GradientOracle):
    """Op = A^-1 through the factors (condest.hpp:138-152); holds them by reference."""

    def __init__(self, factors: LUFactors):
        self.factors = factors

    def dimension(self) -> int:
        return self.factors.n

    def loss(self, x) -> float:
        x = _lib.as_f64(x, self.factors.n)
        out = C.c_double()
        _lib.check(_lib.load().ck_loss_inverse(self.factors.handle, _lib.dptr(x), C.byref(out)),
                   "loss_inverse")
        return out.value

    def grad(self, x) -> np.ndarray:
        x = _lib.as_f64(x, self.factors.n)
        g = np.empty(self.factors.n)
        _lib.check(_lib.load().ck_grad_inverse(self.factors.handle, _lib.dptr(x), _lib.dptr(g)),
                   "grad_inverse")
        return g

    def apply(self, x) -> np.ndarray:
        return self.factors.solve(x)


def grad_inverse(f: LUFactors, x) -> np.ndarray:
    """condest.hpp:112-123."""
    return InverseOracle(f).grad(x)


class InverseSession(Session):
    def __init__(self, oracle: InverseOracle, cfg: AdamConfig, seeds):
        if oracle.dimension() == 0:
            raise InvalidArgument("projected_adam: zero-dimensional operator")
        self.oracle = oracle
        self.n = oracle.dimension()
        lib = _lib.load()
        self._cfg = _lib.cfg_struct(cfg)
        seeds = np.ascontiguousarray([int(s) & 0xFFFFFFFFFFFFFFFF for s in seeds], np.uint64)
        self.ncols = seeds.size
        h = C.c_void_p()
        _lib.check(lib.ck_session_create_inverse(oracle.factors.handle, C.byref(self._cfg),
                                                 seeds.ctypes.data_as(_lib.u64p), self.ncols,
                                                 C.byref(h)), "ck_session_create_inverse")
        self.handle = h
        self._fin = weakref.finalize(self, lib.ck_session_free, h)


def _inverse_projected_adam(oracle: InverseOracle, cfg: AdamConfig, observer):
    from .condest import AdamState, AdamStepInfo  # noqa: PLC0415
    s = InverseSession(oracle, cfg, [cfg.seed])
    try:
        if observer is None:
            s.run()
        else:
            while True:
                info, x, xm = s.step_observed(True)
                if info.phase == 2:
                    break
                observer(AdamState(x=x, t=int(info.t), loss_min=info.loss_min, x_min=xm),
                         AdamStepInfo(info.x_dot_delta, info.delta_norm, info.loss))
        return s.result(0)
    finally:
        s.close()


def _inverse_estimate_norm(oracle: InverseOracle, cfg: AdamConfig, restarts: int):
    r = _lib.NormResult()
    w = np.empty(oracle.dimension())
    c = _lib.cfg_struct(cfg)
    _lib.check(_lib.load().ck_inv_estimate_norm(oracle.factors.handle, C.byref(c), restarts,
                                                C.byref(r), _lib.dptr(w)), "estimate_norm")
    return NormEstimate(r.value, w, int(r.iterations), bool(r.converged))


def inv_norm2(f: LUFactors, cfg: Optional[AdamConfig] = None) -> NormEstimate:
    """||A^-1||_2 estimate, single run (condest.hpp:320-322)."""
    from .condest import projected_adam  # noqa: PLC0415
    return projected_adam(InverseOracle(f), cfg)


@dataclass
class Cond2Result:
    kappa: float = 0.0
    operator_norm: NormEstimate = field(default_factory=NormEstimate)
    inverse_norm: NormEstimate = field(default_factory=NormEstimate)
    factors: Optional[LUFactors] = None


def cond2(a: SparseMatrix, cfg: Optional[AdamConfig] = None, restarts: int = 3,
          pivot_tol: float = 1e-14) -> Cond2Result:
    """kappa_2(A) = ||A|| ||A^-1|| (condest.hpp:341-365); singular -> +inf."""
    cfg = cfg or AdamConfig()
    if a.nrows != a.ncols:
        raise DimensionMismatch("cond2: matrix must be square")
    res = Cond2Result()
    res.operator_norm = estimate_norm(ExplicitOracle(a), cfg, restarts)
    try:
        f = lu_factorize(a, pivot_tol)
    except (StructurallySingular, NumericallySingular):
        res.inverse_norm = NormEstimate(value=math.inf)
        res.kappa = math.inf
        return res
    ci = AdamConfig(**{**cfg.__dict__})
    from .rng import mix_seed  # noqa: PLC0415
    ci.seed = mix_seed(cfg.seed, 0x1234)
    res.inverse_norm = estimate_norm(InverseOracle(f), ci, restarts)
    res.kappa = res.operator_norm.value * res.inverse_norm.value
    res.factors = f
    return res
