"""Projected-Adam norm / condition-number estimation on the B200.

Python mirror of ``condkit/condest.hpp``: same names, argument meaning and
error behaviour. All arithmetic runs in the native library (C-ABI ->
sm_100a kernels); this module only marshals arguments.

Reference map:
  AdamConfig (condest.hpp:39-48), AdamState (:51-56), AdamStepInfo (:61-65),
  NormEstimate (:69-74), GradientOracle (:78-85), ExplicitOracle (:125-135),
  projected_adam (:184-297), estimate_norm (:301-312), norm2 (:315-317).
"""
from __future__ import annotations

import abc
import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from .errors import DegenerateDirection, InvalidArgument
from .sparse import SparseMatrix


@dataclass
class AdamConfig:
    alpha: float = 0.05
    beta1: float = 0.9
    beta2: float = 0.999
    eps_stab: float = 1e-8
    max_iter: int = 2000
    seed: int = 1
    rel_tol: float = 1e-12
    patience: int = 100


@dataclass
class NormEstimate:
    value: float = 0.0
    witness: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterations: int = 0
    converged: bool = False


@dataclass
class AdamState:
    """What the observer sees (condest.hpp:51-56); m and v stay on the device."""
    x: np.ndarray
    t: int
    loss_min: float
    x_min: np.ndarray


@dataclass
class AdamStepInfo:
    x_dot_delta: float = 0.0
    delta_norm: float = 0.0
    loss: float = 0.0


AdamObserver = Callable[[AdamState, AdamStepInfo], None]


class GradientOracle(abc.ABC):
    """L(v) = log||v|| - log||Op v|| (condest.hpp:76-85)."""

    @abc.abstractmethod
    def dimension(self) -> int: ...

    @abc.abstractmethod
    def loss(self, x) -> float: ...

    @abc.abstractmethod
    def grad(self, x) -> np.ndarray: ...

    @abc.abstractmethod
    def apply(self, x) -> np.ndarray: ...


class ExplicitOracle(GradientOracle):
    """Op = A, device resident (condest.hpp:125-135)."""

    def __init__(self, a: SparseMatrix):
        self.a = a

    def dimension(self) -> int:
        return self.a.ncols

    def loss(self, x) -> float:
        x = _lib.as_f64(x, self.a.ncols)
        out = C.c_double()
        _lib.check(_lib.load().ck_loss_explicit(self.a.device().handle, _lib.dptr(x),
                                                C.byref(out)), "loss_explicit")
        return out.value

    def grad(self, x) -> np.ndarray:
        x = _lib.as_f64(x, self.a.ncols)
        g = np.empty(self.a.ncols)
        _lib.check(_lib.load().ck_grad_explicit(self.a.device().handle, _lib.dptr(x),
                                                _lib.dptr(g)), "grad_explicit")
        return g

    def apply(self, x) -> np.ndarray:
        return self.a.device().matvec(x)


def loss_explicit(a: SparseMatrix, v) -> float:
    """condest.hpp:88-93 (raises DegenerateDirection when ||Av|| = 0)."""
    return ExplicitOracle(a).loss(v)


def grad_explicit(a: SparseMatrix, v) -> np.ndarray:
    """condest.hpp:96-107."""
    return ExplicitOracle(a).grad(v)


class Session:
    """Device-resident Projected-Adam loop over ``ncols`` independent seeds."""

    def __init__(self, oracle: GradientOracle, cfg: AdamConfig, seeds):
        if oracle.dimension() == 0:
            raise InvalidArgument("projected_adam: zero-dimensional operator")
        self.oracle = oracle
        self.n = oracle.dimension()
        lib = _lib.load()
        seeds = np.ascontiguousarray([int(s) & 0xFFFFFFFFFFFFFFFF for s in seeds], np.uint64)
        prefetch = (isinstance(oracle, ExplicitOracle) and oracle.a._dev is None and seeds.size
                    and self.n >= (1 << 20))
        if prefetch:
            # draw the first start vector on a host thread while A uploads
            _lib.check(lib.ck_start_vector_prefetch(int(seeds[0]), self.n),
                       "ck_start_vector_prefetch")
        self._cfg = _lib.cfg_struct(cfg)
        self.ncols = seeds.size
        h = C.c_void_p()
        try:
            handle = _device_handle(oracle)
            _lib.check(lib.ck_session_create(handle, C.byref(self._cfg),
                                             seeds.ctypes.data_as(_lib.u64p), self.ncols,
                                             C.byref(h)), "ck_session_create")
        except BaseException:
            if prefetch:  # no session took the slot: release its thread and pinned buffer
                lib.ck_start_vector_prefetch_cancel()
            raise
        self.handle = h
        self._fin = weakref.finalize(self, lib.ck_session_free, h)

    def run(self, max_steps: int = 0) -> bool:
        fin = C.c_int32()
        _lib.check(_lib.load().ck_session_run(self.handle, max_steps, C.byref(fin)),
                   "ck_session_run")
        return bool(fin.value)

    def time(self, steps: int, mode: int = 0):
        tot, a, t = C.c_double(), C.c_double(), C.c_double()
        _lib.check(_lib.load().ck_session_time(self.handle, steps, mode, C.byref(tot), C.byref(a),
                                               C.byref(t)), "ck_session_time")
        return tot.value, a.value, t.value

    def step_observed(self, want_vectors: bool = True):
        info = _lib.StepInfo()
        x = np.empty(self.n) if want_vectors else None
        xm = np.empty(self.n) if want_vectors else None
        _lib.check(_lib.load().ck_session_step_observed(
            self.handle, C.byref(info), _lib.dptr(x) if want_vectors else None,
            _lib.dptr(xm) if want_vectors else None), "ck_session_step_observed")
        return info, x, xm

    def result(self, column: int = 0, witness: bool = True) -> NormEstimate:
        r = _lib.NormResult()
        w = np.empty(self.n) if witness else None
        _lib.check(_lib.load().ck_session_result(self.handle, column, C.byref(r),
                                                 _lib.dptr(w) if witness else None),
                   "ck_session_result")
        return NormEstimate(r.value, w if witness else np.zeros(0), int(r.iterations),
                            bool(r.converged))

    def close(self) -> None:
        self._fin()


def _device_handle(oracle: GradientOracle):
    if isinstance(oracle, ExplicitOracle):
        return oracle.a.device().handle
    raise TypeError(f"{type(oracle).__name__}: only device oracles are supported "
                    "(ExplicitOracle, InverseOracle); there is no host fallback")


def projected_adam(oracle: GradientOracle, cfg: Optional[AdamConfig] = None,
                   observer: Optional[AdamObserver] = None) -> NormEstimate:
    """Minimise L over the unit sphere (condest.hpp:184-297)."""
    cfg = cfg or AdamConfig()
    from .inverse import InverseOracle, _inverse_projected_adam  # noqa: PLC0415
    if isinstance(oracle, InverseOracle):
        return _inverse_projected_adam(oracle, cfg, observer)
    s = Session(oracle, cfg, [cfg.seed])
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


def estimate_norm(oracle: GradientOracle, cfg: Optional[AdamConfig] = None,
                  restarts: int = 3) -> NormEstimate:
    """Best of `restarts` seeded runs (condest.hpp:301-312)."""
    cfg = cfg or AdamConfig()
    if restarts == 0:
        raise InvalidArgument("estimate_norm: restarts must be >= 1")
    from .inverse import InverseOracle, _inverse_estimate_norm  # noqa: PLC0415
    if isinstance(oracle, InverseOracle):
        return _inverse_estimate_norm(oracle, cfg, restarts)
    if not isinstance(oracle, ExplicitOracle):
        _device_handle(oracle)
    r = _lib.NormResult()
    w = np.empty(oracle.dimension())
    c = _lib.cfg_struct(cfg)
    _lib.check(_lib.load().ck_estimate_norm(oracle.a.device().handle, C.byref(c), restarts,
                                            C.byref(r), _lib.dptr(w)), "estimate_norm")
    return NormEstimate(r.value, w, int(r.iterations), bool(r.converged))


def norm2(a: SparseMatrix, cfg: Optional[AdamConfig] = None) -> NormEstimate:
    """||A||_2 estimate, single run (condest.hpp:315-317)."""
    return projected_adam(ExplicitOracle(a), cfg)


__all__ = ["AdamConfig", "AdamState", "AdamStepInfo", "NormEstimate", "GradientOracle",
           "ExplicitOracle", "Session", "projected_adam", "estimate_norm", "norm2",
           "loss_explicit", "grad_explicit", "DegenerateDirection"]
