"""Forward-error bounds driven by kappa_2 (mirror of condkit/error_bounds.hpp).

The scalar formulas run in the native library (ck_loose_bounds etc.); the
residual ||A x^ - b|| and the norms run on the device; kappa and ||A|| come
from the device estimator (cond2 / estimate_norm).

Reference map: kEpsMach (error_bounds.hpp:31), loose_bounds (:59-68),
tight_bounds (:71-80), propagate_bound (:84-88), singularity_bound (:93-99),
Verdict (:101-110), BoundsReport (:112-147), VerifyOptions (:149-157),
verify_solution (:166-217).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

from . import _lib
from .condest import AdamConfig
from .errors import DimensionMismatch, InvalidArgument, ZeroRHS, ZeroSolution

kEpsMach = 2.0 ** -53


@dataclass(frozen=True)
class Bounds:
    lower: float = 0.0
    upper: float = 0.0


def _pair(fn, *args):
    lo, hi = C.c_double(), C.c_double()
    _lib.check(fn(*args, C.byref(lo), C.byref(hi)), fn.__name__)
    return Bounds(lo.value, hi.value)


def loose_bounds(residual_norm: float, b_norm: float, kappa: float) -> Bounds:
    return _pair(_lib.load().ck_loose_bounds, residual_norm, b_norm, kappa)


def tight_bounds(residual_norm: float, a_norm: float, xhat_norm: float, kappa: float) -> Bounds:
    return _pair(_lib.load().ck_tight_bounds, residual_norm, a_norm, xhat_norm, kappa)


def propagate_bound(eps_tight: float) -> float:
    out = C.c_double()
    _lib.check(_lib.load().ck_propagate_bound(eps_tight, C.byref(out)), "propagate_bound")
    return out.value


def singularity_bound(kappa: float, eps_mach: float = kEpsMach) -> float:
    out = C.c_double()
    _lib.check(_lib.load().ck_singularity_bound(kappa, eps_mach, C.byref(out)),
               "singularity_bound")
    return out.value


class Verdict(enum.IntEnum):
    accepted = 0
    rejected = 1
    numerically_singular = 2


def _fmt17(v: float) -> str:
    """format_significant17 (format.hpp:10-14): shortest-of-17-significant-digits."""
    s = f"{v:.17g}"
    if s in ("inf", "-inf", "nan"):
        return s
    return s


@dataclass
class BoundsReport:
    residual_norm: float = 0.0
    b_norm: float = 0.0
    a_norm: float = 0.0
    xhat_norm: float = 0.0
    kappa: float = 0.0
    kappa_supplied: bool = False
    loose_lower: float = 0.0
    loose_upper: float = 0.0
    tight_lower: float = 0.0
    tight_upper: float = 0.0
    true_error_cap: float = 0.0
    singularity_cap: float = 0.0
    threshold: float = 0.0
    eps_mach: float = kEpsMach
    verdict: Verdict = Verdict.rejected

    def to_kv(self):
        f = _fmt17
        return [("residual_norm", f(self.residual_norm)), ("b_norm", f(self.b_norm)),
                ("a_norm", f(self.a_norm)), ("xhat_norm", f(self.xhat_norm)),
                ("kappa", f(self.kappa)),
                ("kappa_source", "supplied" if self.kappa_supplied else "estimated"),
                ("loose_lower", f(self.loose_lower)), ("loose_upper", f(self.loose_upper)),
                ("tight_lower", f(self.tight_lower)), ("tight_upper", f(self.tight_upper)),
                ("true_error_cap", f(self.true_error_cap)),
                ("singularity_cap", f(self.singularity_cap)), ("threshold", f(self.threshold)),
                ("eps_mach", f(self.eps_mach)), ("verdict", self.verdict.name)]


@dataclass
class VerifyOptions:
    threshold: float = 1e-7
    kappa: Optional[float] = None
    a_norm: Optional[float] = None
    eps_mach: float = kEpsMach
    adam: AdamConfig = field(default_factory=AdamConfig)
    restarts: int = 3
    pivot_tol: float = 1e-14


def verify_solution(a, xhat, b, opt: Optional[VerifyOptions] = None) -> BoundsReport:
    """Fill a BoundsReport for (A, x^, b) (error_bounds.hpp:166-217)."""
    from .condest import ExplicitOracle, estimate_norm  # noqa: PLC0415
    opt = opt or VerifyOptions()
    if a.nrows != a.ncols:
        raise DimensionMismatch("verify_solution: matrix must be square")
    if len(xhat) != a.ncols:
        raise DimensionMismatch("verify_solution: solution length")
    if len(b) != a.nrows:
        raise DimensionMismatch("verify_solution: rhs length")
    if not opt.threshold > 0.0:
        raise InvalidArgument("threshold must be > 0")
    rep = BoundsReport(threshold=opt.threshold, eps_mach=opt.eps_mach)
    rn, xn, bn = a.device().residual_norms(xhat, b)
    rep.xhat_norm = xn
    if xn == 0.0:
        raise ZeroSolution("candidate solution has zero norm")
    rep.b_norm = bn
    if bn == 0.0:
        raise ZeroRHS("right-hand side has zero norm")
    rep.residual_norm = rn
    if opt.kappa is not None:
        if not opt.kappa >= 1.0:
            raise InvalidArgument("kappa must be >= 1")
        rep.kappa, rep.kappa_supplied = opt.kappa, True
        rep.a_norm = (opt.a_norm if opt.a_norm is not None
                      else estimate_norm(ExplicitOracle(a), opt.adam, opt.restarts).value)
    else:
        from .inverse import cond2  # noqa: PLC0415
        c = cond2(a, opt.adam, opt.restarts, opt.pivot_tol)
        rep.kappa = max(1.0, c.kappa)
        rep.a_norm = opt.a_norm if opt.a_norm is not None else c.operator_norm.value
    if not rep.a_norm > 0.0:
        raise InvalidArgument("operator norm must be > 0")
    lb = loose_bounds(rep.residual_norm, rep.b_norm, rep.kappa)
    rep.loose_lower, rep.loose_upper = lb.lower, lb.upper
    tb = tight_bounds(rep.residual_norm, rep.a_norm, rep.xhat_norm, rep.kappa)
    rep.tight_lower, rep.tight_upper = tb.lower, tb.upper
    rep.true_error_cap = propagate_bound(rep.tight_upper)
    rep.singularity_cap = singularity_bound(rep.kappa, rep.eps_mach)
    if rep.kappa >= 1.0 / rep.eps_mach:
        rep.verdict = Verdict.numerically_singular
    else:
        rep.verdict = Verdict.accepted if rep.tight_upper <= rep.threshold else Verdict.rejected
    return rep
