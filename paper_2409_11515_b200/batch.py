"""Batched ensembles (BASELINE config 5): many independent matrices, several
restarts each, advanced together by one kernel pair per iteration.

The members are packed block-diagonally into one device operator, each member
tile-aligned (padded to a multiple of 256 rows/columns with empty rows). Every
member keeps its own control state, RNG streams, restarts and result; the
arithmetic of a member is the same as running it alone.
"""
from __future__ import annotations

import ctypes as C
import weakref
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .condest import AdamConfig, NormEstimate, Session
from .errors import NumericallySingular, StructurallySingular
from .rng import mix_seed
from .sparse import SparseMatrix

TILE = 256


def pack_block_diagonal(members: Sequence[SparseMatrix]):
    """(packed SparseMatrix, seg_n) with member g at offset sum(round_up(n_h, 256))."""
    offs, rps, cis, vas = [], [], [], []
    off = 0
    nnz = 0
    for m in members:
        if m.nrows != m.ncols:
            raise ValueError("batched members must be square")
        pad = -(-m.nrows // TILE) * TILE
        rp = m.row_offsets[1:] + nnz
        rps.append(rp)
        rps.append(np.full(pad - m.nrows, rp[-1] if rp.size else nnz, np.int64))
        cis.append(m.col_indices.astype(np.int64) + off)
        vas.append(m.values)
        offs.append(off)
        off += pad
        nnz += m.nnz
    rp = np.concatenate([np.zeros(1, np.int64)] + rps)
    ci = np.concatenate(cis).astype(np.int32)
    va = np.concatenate(vas)
    packed = SparseMatrix(off, off, rp, ci, va, validate=False)
    return packed, np.array([m.nrows for m in members], np.int64)


def member_seeds(count: int, seed: int = 1) -> list[int]:
    """Per-member estimator seeds, as run_bench seeds cond2 per matrix (bench.hpp:435)."""
    return [mix_seed(seed, 0x1000 + m) for m in range(count)]


def estimate_norm_batch(members: Sequence[SparseMatrix], cfg: Optional[AdamConfig] = None,
                        restarts: int = 4, seeds: Optional[Sequence[int]] = None,
                        packed=None) -> list[NormEstimate]:
    """estimate_norm (condest.hpp:301-312) for every member, all on one device sweep."""
    cfg = cfg or AdamConfig()
    if packed is None:
        packed = pack_block_diagonal(members)
    a, seg_n = packed
    seeds = np.ascontiguousarray(seeds if seeds is not None else [cfg.seed] * seg_n.size,
                                 np.uint64)
    res = (_lib.NormResult * seg_n.size)()
    c = _lib.cfg_struct(cfg)
    _lib.check(_lib.load().ck_estimate_norm_batch(
        a.device().handle, seg_n.ctypes.data_as(_lib.i64p), int(seg_n.size), C.byref(c),
        seeds.ctypes.data_as(_lib.u64p), restarts, res), "estimate_norm_batch")
    return [NormEstimate(r.value, np.zeros(0), int(r.iterations), bool(r.converged)) for r in res]


class BatchSession(Session):
    """Device loop over a packed batch: members x restart columns (bench / inspection)."""

    def __init__(self, packed, cfg: AdamConfig, seeds_per_member_column):
        a, seg_n = packed
        self.oracle = a  # keeps the device matrix alive
        self.seg_n = seg_n
        self.n = int(seg_n.max())
        seeds = np.ascontiguousarray(seeds_per_member_column, np.uint64)
        self.ncols = seeds.size // seg_n.size
        lib = _lib.load()
        self._cfg = _lib.cfg_struct(cfg)
        h = C.c_void_p()
        _lib.check(lib.ck_session_create_batch(a.device().handle, seg_n.ctypes.data_as(_lib.i64p),
                                               int(seg_n.size), C.byref(self._cfg),
                                               seeds.ctypes.data_as(_lib.u64p), self.ncols,
                                               C.byref(h)), "ck_session_create_batch")
        self.handle = h
        self._fin = weakref.finalize(self, lib.ck_session_free, h)

    def member_result(self, g: int, c: int = 0) -> NormEstimate:
        r = _lib.NormResult()
        w = np.empty(int(self.seg_n[g]))
        _lib.check(_lib.load().ck_session_result(self.handle, g * self.ncols + c, C.byref(r),
                                                 _lib.dptr(w)), "ck_session_result")
        return NormEstimate(r.value, w, int(r.iterations), bool(r.converged))


# ------------------------------------------------------------ sigma_min side
def lu_factorize_many(members: Sequence[SparseMatrix], pivot_tol: float = 1e-14,
                      threads: int = 8) -> list:
    """lu_factorize for every member in one batched device factorisation
    (ck_lu_factorize_batch: one panel loop for all members). Singular members
    give the exception instance instead of factors. `threads` is kept for
    compatibility (the device batch needs none)."""
    from .errors import from_status  # noqa: PLC0415
    from .inverse import LUFactors  # noqa: PLC0415
    del threads
    if not members:
        return []
    lib = _lib.load()
    S = len(members)
    hs = (C.c_void_p * S)()
    for g, m in enumerate(members):
        hs[g] = m.device().handle
    out = (C.c_void_p * S)()
    status = np.zeros(S, np.int32)
    fcol = np.zeros(S, np.int64)
    fpiv = np.zeros(S)
    _lib.check(lib.ck_lu_factorize_batch(C.cast(hs, C.c_void_p), S, pivot_tol, C.cast(out, C.c_void_p),
                                         _lib.i32ptr(status), fcol.ctypes.data_as(_lib.i64p),
                                         _lib.dptr(fpiv)), "ck_lu_factorize_batch")
    res = []
    for g, m in enumerate(members):
        if status[g] == 0:
            res.append(LUFactors(C.c_void_p(out[g]), m.nrows))
        else:
            e = from_status(int(status[g]), f"lu_factorize: member {g}: column {int(fcol[g])}, "
                                            f"pivot {float(fpiv[g]):.3e}")
            if not isinstance(e, (StructurallySingular, NumericallySingular)):
                raise e
            res.append(e)
    return res


def _lu_handles(factors):
    arr = (C.c_void_p * len(factors))()
    for g, f in enumerate(factors):
        arr[g] = f.handle
    return arr


def inv_estimate_norm_batch(factors, cfg: Optional[AdamConfig] = None, restarts: int = 4,
                            seeds: Optional[Sequence[int]] = None) -> list[NormEstimate]:
    """estimate_norm on A_g^-1 (InverseOracle, condest.hpp:156-175, 301-312) for
    every member, one device CTA per member per step."""
    cfg = cfg or AdamConfig()
    seeds = np.ascontiguousarray(seeds if seeds is not None else [cfg.seed] * len(factors),
                                 np.uint64)
    res = (_lib.NormResult * len(factors))()
    c = _lib.cfg_struct(cfg)
    _lib.check(_lib.load().ck_inv_estimate_norm_batch(
        _lu_handles(factors), len(factors), C.byref(c), seeds.ctypes.data_as(_lib.u64p), restarts,
        res), "inv_estimate_norm_batch")
    return [NormEstimate(r.value, np.zeros(0), int(r.iterations), bool(r.converged)) for r in res]


class InverseBatchSession(Session):
    """Device loop over many factorisations: members x restart columns."""

    def __init__(self, factors, cfg: AdamConfig, seeds_per_member_column):
        self.factors = list(factors)  # keeps the factors alive
        self.seg_n = np.array([f.n for f in self.factors], np.int64)
        self.n = int(self.seg_n.max())
        seeds = np.ascontiguousarray(seeds_per_member_column, np.uint64)
        self.ncols = seeds.size // len(self.factors)
        lib = _lib.load()
        self._cfg = _lib.cfg_struct(cfg)
        h = C.c_void_p()
        _lib.check(lib.ck_session_create_inverse_batch(
            _lu_handles(self.factors), len(self.factors), C.byref(self._cfg),
            seeds.ctypes.data_as(_lib.u64p), self.ncols, C.byref(h)),
            "ck_session_create_inverse_batch")
        self.handle = h
        self._fin = weakref.finalize(self, lib.ck_session_free, h)

    def member_result(self, g: int, c: int = 0) -> NormEstimate:
        r = _lib.NormResult()
        w = np.empty(int(self.seg_n[g]))
        _lib.check(_lib.load().ck_session_result(self.handle, g * self.ncols + c, C.byref(r),
                                                 _lib.dptr(w)), "ck_session_result")
        return NormEstimate(r.value, w, int(r.iterations), bool(r.converged))


def _band_bytes(a: SparseMatrix) -> int:
    """Device bytes of a's band LU (lu.hpp layout, ldab = 2 kl + ku + 1) plus the
    solve working vectors, from the CSR's band."""
    rp, ci = a.row_offsets, a.col_indices
    rows = np.repeat(np.arange(a.nrows, dtype=np.int64), np.diff(rp))
    d = rows - ci.astype(np.int64)
    kl = int(d.max(initial=0))
    ku = int((-d).max(initial=0))
    return 8 * a.nrows * (2 * kl + ku + 1 + 64) + (1 << 20)


def auto_wave(members: Sequence[SparseMatrix], fraction: float = 0.7) -> int:
    """Members factorised and iterated at once: one CTA each, so up to the SM
    count (config 5: 64 -> 148 members lifts sigma_min throughput 1917 -> 4433
    run-iterations/s, scripts/time_inverse_batch.py), bounded by `fraction` of
    the free device memory for the band LUs."""
    free, total, sms = C.c_uint64(0), C.c_uint64(0), C.c_int32(0)
    _lib.check(_lib.load().ck_device_memory(C.byref(free), C.byref(total), C.byref(sms)),
               "ck_device_memory")
    per = max(_band_bytes(m) for m in members) if members else 1
    return max(1, min(int(sms.value), int(fraction * free.value) // per))


def cond2_batch(members: Sequence[SparseMatrix], cfg: Optional[AdamConfig] = None,
                restarts: int = 4, pivot_tol: float = 1e-14,
                seeds: Optional[Sequence[int]] = None, wave: Optional[int] = None,
                threads: int = 8):
    """cond2 (condest.hpp:341-365) of every member, as run_bench computes it per
    matrix with seed seeds[g] (default: member_seeds): ||A_g|| for the whole
    ensemble in one packed device sweep, then the factorisations and ||A_g^-1||
    in waves of `wave` members (default auto_wave: as many as SMs, within the
    device memory), one CTA per member."""
    from .inverse import Cond2Result  # noqa: PLC0415
    cfg = cfg or AdamConfig()
    seeds = list(seeds) if seeds is not None else member_seeds(len(members), cfg.seed)
    fwd = estimate_norm_batch(members, cfg, restarts, seeds)
    if wave is None:
        wave = auto_wave(members)
    out = [Cond2Result(operator_norm=e) for e in fwd]
    for w0 in range(0, len(members), wave):
        idx = list(range(w0, min(len(members), w0 + wave)))
        facs = lu_factorize_many([members[g] for g in idx], pivot_tol, threads)
        ok = [g for g, f in zip(idx, facs) if not isinstance(f, Exception)]
        for g, f in zip(idx, facs):
            if isinstance(f, Exception):
                out[g].inverse_norm = NormEstimate(value=float("inf"))
                out[g].kappa = float("inf")
        if ok:
            fs = [facs[g - w0] for g in ok]
            inv = inv_estimate_norm_batch(fs, cfg, restarts,
                                          [mix_seed(seeds[g], 0x1234) for g in ok])
            for g, e in zip(ok, inv):
                out[g].inverse_norm = e
                out[g].kappa = out[g].operator_norm.value * e.value
        del facs
    return out
