"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU oracles.

Two interchangeable backends with identical signatures:
  * ``Oracle("port")`` -> oracle/_build/libcondkit_oracle.so, the plain-C restatement
    (oracle/condkit_oracle.c) of the reference path;
  * ``Oracle("ref")``  -> oracle/_ref/libcondkit_ref.so, the unmodified reference
    headers compiled in place (oracle/ref_driver.cpp), only where it was built.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference
arm may import this module. The product package never does.

Matrices are duck-typed: any object with ``nrows``, ``ncols``, ``row_offsets``
(int64), ``col_indices`` (int32) and ``values`` (float64) works; configs need
the ``AdamConfig`` attribute names of condest.hpp:39-48.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": os.path.join(HERE, "_build", "libcondkit_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libcondkit_ref.so"),
    # the same reference driver at -O3, for bench.py's CPU arms
    "ref_v3": os.path.join(HERE, "_ref", "libcondkit_ref_v3.so"),
    "ref_native": os.path.join(HERE, "_ref", "libcondkit_ref_native.so"),
}
PREFIX = {"port": "cko_", "ref": "ckref_", "ref_v3": "ckref_", "ref_native": "ckref_"}
BUILD_FLAGS = {
    "port": "gcc -O2 -ffp-contract=off (C restatement)",
    "ref": "g++ -O2 -ffp-contract=off -std=c++20",
    "ref_v3": "g++ -O3 -march=x86-64-v3 -ffp-contract=off -std=c++20",
    "ref_native": "g++ -O3 -march=native (Sapphire Rapids build host) -ffp-contract=off -std=c++20",
}
GEN_PATH = os.path.join(HERE, "_build", "libcondkit_gen.so")


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def best_reference() -> str:
    """The fastest reference build this host can execute: the -march=native build only
    where every ISA extension of its build host is present, else -O3 x86-64-v3, else -O2."""
    flags = _cpu_flags()
    isa = os.path.join(HERE, "_ref", "native_isa.txt")
    if available("ref_native") and os.path.exists(isa):
        with open(isa) as f:
            need = {w.strip() for w in f if w.strip()}
        if need and need <= flags:
            return "ref_native"
    if available("ref_v3") and {"avx2", "fma", "bmi2"} <= flags:
        return "ref_v3"
    return "ref" if available("ref") else "port"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


@dataclass
class CSR:
    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])


def generate(kind: int, grid: int, seed: int = 1, param: int = 0) -> CSR:
    """The BASELINE synthetic operators from _build/libcondkit_gen.so,
    a g++ build of the product's host generator source: bench.py's reference arm builds its
    workload with this instead of loading libcondkit_b200.so."""
    lib = C.CDLL(GEN_PATH)
    f = lib.ck_generate
    f.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_uint64, _i64p, _i64p, _i64p, _i32p, _dp]
    f.restype = C.c_int
    n, nnz = C.c_int64(), C.c_int64()
    if f(kind, grid, param, seed, C.byref(n), C.byref(nnz), None, None, None):
        raise OracleError(2, "ck_generate(size)")
    rp = np.empty(n.value + 1, np.int64)
    ci = np.empty(max(nnz.value, 1), np.int32)
    va = np.empty(max(nnz.value, 1), np.float64)
    if f(kind, grid, param, seed, C.byref(n), C.byref(nnz), rp.ctypes.data_as(_i64p),
         ci.ctypes.data_as(_i32p), va.ctypes.data_as(_dp)):
        raise OracleError(2, "ck_generate")
    return CSR(n.value, n.value, rp, ci[: nnz.value], va[: nnz.value])

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)


class AdamCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps_stab", C.c_double), ("max_iter", C.c_uint64), ("seed", C.c_uint64),
                ("rel_tol", C.c_double), ("patience", C.c_uint64)]


class NormRes(C.Structure):
    _fields_ = [("value", C.c_double), ("iterations", C.c_uint64), ("converged", C.c_int32),
                ("_pad", C.c_int32)]


class BoundsRep(C.Structure):
    _fields_ = [("residual_norm", C.c_double), ("b_norm", C.c_double), ("a_norm", C.c_double),
                ("xhat_norm", C.c_double), ("kappa", C.c_double), ("kappa_supplied", C.c_int32),
                ("verdict", C.c_int32), ("loose_lower", C.c_double), ("loose_upper", C.c_double),
                ("tight_lower", C.c_double), ("tight_upper", C.c_double),
                ("true_error_cap", C.c_double), ("singularity_cap", C.c_double),
                ("threshold", C.c_double), ("eps_mach", C.c_double)]


class VerifyOpts(C.Structure):
    _fields_ = [("threshold", C.c_double), ("has_kappa", C.c_int32), ("has_a_norm", C.c_int32),
                ("kappa", C.c_double), ("a_norm", C.c_double), ("eps_mach", C.c_double),
                ("adam", AdamCfg), ("restarts", C.c_uint64), ("pivot_tol", C.c_double)]


@dataclass
class Estimate:
    value: float
    iterations: int
    converged: bool
    witness: np.ndarray | None = None
    trace: np.ndarray | None = None


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: status {code}")
        self.code = code


def _d(a):
    return a.ctypes.data_as(_dp)


def _cfg(cfg) -> AdamCfg:
    return AdamCfg(cfg.alpha, cfg.beta1, cfg.beta2, cfg.eps_stab, int(cfg.max_iter),
                   int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, cfg.rel_tol, int(cfg.patience))


def _csr(a):
    rp = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_indices, dtype=np.int32)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    return (int(a.nrows), int(a.ncols), rp, ci, va)


def available(which: str) -> bool:
    return os.path.exists(PATHS[which])


class LUHandle:
    def __init__(self, owner: "Oracle", ptr):
        self._o, self.ptr = owner, ptr
        n, nl, nu, pm = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        owner._f("lu_info")(ptr, C.byref(n), C.byref(nl), C.byref(nu), C.byref(pm))
        self.n, self.nnz_l, self.nnz_u, self.pivot_min = n.value, nl.value, nu.value, pm.value

    def export(self):
        n = self.n
        lrp, urp = np.zeros(n + 1, np.int64), np.zeros(n + 1, np.int64)
        lci, uci = np.zeros(max(self.nnz_l, 1), np.int32), np.zeros(max(self.nnz_u, 1), np.int32)
        lva, uva = np.zeros(max(self.nnz_l, 1)), np.zeros(max(self.nnz_u, 1))
        perm = np.zeros(n, np.int64)
        self._o._f("lu_export")(self.ptr, lrp.ctypes.data_as(_i64p), lci.ctypes.data_as(_i32p),
                                _d(lva), urp.ctypes.data_as(_i64p), uci.ctypes.data_as(_i32p),
                                _d(uva), perm.ctypes.data_as(_i64p))
        return dict(l=(lrp, lci[: self.nnz_l], lva[: self.nnz_l]),
                    u=(urp, uci[: self.nnz_u], uva[: self.nnz_u]), row_perm=perm)

    def __del__(self):
        try:
            self._o._f("lu_free")(self.ptr)
        except Exception:
            pass


class Oracle:
    def __init__(self, which: str = "port"):
        if not available(which):
            raise FileNotFoundError(f"oracle backend '{which}' not built: {PATHS[which]}")
        self.which = which
        self.lib = C.CDLL(PATHS[which])
        self.p = PREFIX[which]
        f = self._f
        f("two_norm").restype = C.c_double
        f("dot").restype = C.c_double
        f("compensated_norm").restype = C.c_double
        f("mix_seed").restype = C.c_uint64
        f("mix_seed").argtypes = [C.c_uint64, C.c_uint64]
        for name in ("loose_bounds", "tight_bounds", "propagate_bound", "singularity_bound"):
            f(name).restype = C.c_int
        f("lu_factorize").argtypes = [C.c_int64, _i64p, _i32p, _dp, C.c_double,
                                      C.POINTER(C.c_void_p), _i64p, _dp]
        f("lu_info").argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _dp]
        f("lu_free").argtypes = [C.c_void_p]
        for name in ("lu_solve", "lu_transpose_solve", "loss_inverse", "grad_inverse"):
            f(name).argtypes = [C.c_void_p, _dp, _dp]
        f("lu_export").argtypes = [C.c_void_p] + [_i64p, _i32p, _dp] * 2 + [_i64p]
        f("projected_adam_inverse").argtypes = [C.c_void_p, C.POINTER(AdamCfg),
                                                C.POINTER(NormRes), _dp, _dp]
        f("estimate_norm_inverse").argtypes = [C.c_void_p, C.POINTER(AdamCfg), C.c_uint64,
                                               C.POINTER(NormRes), _dp]

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    # rng.hpp
    def mix_seed(self, base: int, stream: int) -> int:
        return int(self._f("mix_seed")(base & (2**64 - 1), stream & (2**64 - 1)))

    def mt_draws(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.uint64)
        self._f("mt_draws")(C.c_uint64(seed), C.c_int64(count), out.ctypes.data_as(_u64p))
        return out

    def random_unit_vectors(self, seed: int, n: int, count: int = 1) -> np.ndarray:
        out = np.zeros((count, n))
        self._f("random_unit_vectors")(C.c_uint64(seed), C.c_int64(n), C.c_int64(count), _d(out))
        return out

    def uniform_in(self, seed: int, count: int, lo: float, hi: float) -> np.ndarray:
        out = np.zeros(count)
        self._f("uniform_in")(C.c_uint64(seed), C.c_int64(count), C.c_double(lo), C.c_double(hi),
                              _d(out))
        return out

    # sparse.hpp
    def two_norm(self, v) -> float:
        v = np.ascontiguousarray(v, np.float64)
        return self._f("two_norm")(C.c_int64(v.size), _d(v))

    def dot(self, a, b) -> float:
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        return self._f("dot")(C.c_int64(a.size), _d(a), _d(b))

    def compensated_norm(self, v) -> float:
        v = np.ascontiguousarray(v, np.float64)
        return self._f("compensated_norm")(C.c_int64(v.size), _d(v))

    def matvec(self, a, x) -> np.ndarray:
        nr, nc, rp, ci, va = _csr(a)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(nr)
        self._f("matvec")(C.c_int64(nr), C.c_int64(nc), rp.ctypes.data_as(_i64p),
                          ci.ctypes.data_as(_i32p), _d(va), _d(x), _d(y))
        return y

    def generate_illconditioned(self, n: int, seed: int):
        """Reference only: bench.hpp generate_illconditioned (default spec) as CSR."""
        f = self._f("generate_illconditioned")
        f.restype = C.c_int64
        nnz = f(C.c_int64(n), C.c_uint64(seed), None, None, None)
        rp, ci, va = np.zeros(n + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
        f(C.c_int64(n), C.c_uint64(seed), rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i32p), _d(va))
        return n, rp, ci, va

    def read_matrix_market(self, path: str):
        """Reference only: read_matrix_market of a file -> (nrows, ncols, rp, ci, va) or None."""
        f = self._f("read_matrix_market")
        f.restype = C.c_int64
        nr, nc = C.c_int64(), C.c_int64()
        nnz = f(path.encode(), C.byref(nr), C.byref(nc), None, None, None)
        if nnz < 0:
            return None
        rp, ci, va = np.zeros(nr.value + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
        f(path.encode(), C.byref(nr), C.byref(nc), rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i32p),
          _d(va))
        return nr.value, nc.value, rp, ci, va

    def column_norms(self, a) -> np.ndarray:
        nr, nc, rp, ci, va = _csr(a)
        out = np.zeros(nc)
        self._f("column_norms")(C.c_int64(nr), C.c_int64(nc), rp.ctypes.data_as(_i64p),
                                ci.ctypes.data_as(_i32p), _d(va), _d(out))
        return out

    def row_norms(self, a) -> np.ndarray:
        nr, nc, rp, ci, va = _csr(a)
        out = np.zeros(nr)
        self._f("row_norms")(C.c_int64(nr), rp.ctypes.data_as(_i64p), _d(va), _d(out))
        return out

    def transpose_matvec(self, a, x) -> np.ndarray:
        nr, nc, rp, ci, va = _csr(a)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(nc)
        self._f("transpose_matvec")(C.c_int64(nr), C.c_int64(nc), rp.ctypes.data_as(_i64p),
                                    ci.ctypes.data_as(_i32p), _d(va), _d(x), _d(y))
        return y

    # condest.hpp (explicit)
    def _csr_args(self, a):
        nr, nc, rp, ci, va = _csr(a)
        return (nr, nc, rp, ci, va), (C.c_int64(nr), C.c_int64(nc), rp.ctypes.data_as(_i64p),
                                      ci.ctypes.data_as(_i32p), _d(va))

    def loss_explicit(self, a, x):
        keep, args = self._csr_args(a)
        x = np.ascontiguousarray(x, np.float64)
        out = C.c_double()
        st = self._f("loss_explicit")(*args, _d(x), C.byref(out))
        if st:
            raise OracleError(st, "loss_explicit")
        return out.value

    def grad_explicit(self, a, x):
        keep, args = self._csr_args(a)
        x = np.ascontiguousarray(x, np.float64)
        g = np.zeros(keep[1])
        st = self._f("grad_explicit")(*args, _d(x), _d(g))
        if st:
            raise OracleError(st, "grad_explicit")
        return g

    def projected_adam_explicit(self, a, cfg, trace: bool = False) -> Estimate:
        keep, args = self._csr_args(a)
        c, r = _cfg(cfg), NormRes()
        w = np.zeros(keep[1])
        tr = np.zeros(max(int(cfg.max_iter), 1)) if trace else None
        st = self._f("projected_adam_explicit")(*args, C.byref(c), C.byref(r), _d(w),
                                                _d(tr) if trace else None)
        if st:
            raise OracleError(st, "projected_adam_explicit")
        return Estimate(r.value, r.iterations, bool(r.converged), w, tr)

    def estimate_norm_explicit(self, a, cfg, restarts: int = 3) -> Estimate:
        keep, args = self._csr_args(a)
        c, r = _cfg(cfg), NormRes()
        w = np.zeros(keep[1])
        st = self._f("estimate_norm_explicit")(*args, C.byref(c), C.c_uint64(restarts),
                                               C.byref(r), _d(w))
        if st:
            raise OracleError(st, "estimate_norm_explicit")
        return Estimate(r.value, r.iterations, bool(r.converged), w)

    # lu.hpp
    def lu_factorize(self, a, pivot_tol: float = 1e-12) -> LUHandle:
        nr, nc, rp, ci, va = _csr(a)
        ptr = C.c_void_p()
        col, piv = C.c_int64(-1), C.c_double(0.0)
        st = self._f("lu_factorize")(C.c_int64(nr), rp.ctypes.data_as(_i64p),
                                     ci.ctypes.data_as(_i32p), _d(va), C.c_double(pivot_tol),
                                     C.byref(ptr), C.byref(col), C.byref(piv))
        if st:
            e = OracleError(st, "lu_factorize")
            e.column, e.pivot = col.value, piv.value
            raise e
        return LUHandle(self, ptr)

    def lu_solve(self, f: LUHandle, b) -> np.ndarray:
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(f.n)
        self._f("lu_solve")(f.ptr, _d(b), _d(x))
        return x

    def lu_transpose_solve(self, f: LUHandle, b) -> np.ndarray:
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(f.n)
        self._f("lu_transpose_solve")(f.ptr, _d(b), _d(x))
        return x

    def loss_inverse(self, f: LUHandle, x) -> float:
        x = np.ascontiguousarray(x, np.float64)
        out = C.c_double()
        st = self._f("loss_inverse")(f.ptr, _d(x), C.cast(C.pointer(out), _dp))
        if st:
            raise OracleError(st, "loss_inverse")
        return out.value

    def grad_inverse(self, f: LUHandle, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        g = np.zeros(f.n)
        st = self._f("grad_inverse")(f.ptr, _d(x), _d(g))
        if st:
            raise OracleError(st, "grad_inverse")
        return g

    def projected_adam_inverse(self, f: LUHandle, cfg, trace: bool = False) -> Estimate:
        c, r = _cfg(cfg), NormRes()
        w = np.zeros(f.n)
        tr = np.zeros(max(int(cfg.max_iter), 1)) if trace else None
        st = self._f("projected_adam_inverse")(f.ptr, C.byref(c), C.byref(r), _d(w),
                                               _d(tr) if trace else None)
        if st:
            raise OracleError(st, "projected_adam_inverse")
        return Estimate(r.value, r.iterations, bool(r.converged), w, tr)

    def estimate_norm_inverse(self, f: LUHandle, cfg, restarts: int = 3) -> Estimate:
        c, r = _cfg(cfg), NormRes()
        w = np.zeros(f.n)
        st = self._f("estimate_norm_inverse")(f.ptr, C.byref(c), C.c_uint64(restarts),
                                              C.byref(r), _d(w))
        if st:
            raise OracleError(st, "estimate_norm_inverse")
        return Estimate(r.value, r.iterations, bool(r.converged), w)

    def cond2(self, a, cfg, restarts: int = 3, pivot_tol: float = 1e-14):
        nr, nc, rp, ci, va = _csr(a)
        c = _cfg(cfg)
        kappa, fwd, inv, hf = C.c_double(), NormRes(), NormRes(), C.c_int32()
        st = self._f("cond2")(C.c_int64(nr), rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i32p),
                              _d(va), C.byref(c), C.c_uint64(restarts), C.c_double(pivot_tol),
                              C.byref(kappa), C.byref(fwd), C.byref(inv), C.byref(hf))
        if st:
            raise OracleError(st, "cond2")
        return dict(kappa=kappa.value,
                    operator_norm=Estimate(fwd.value, fwd.iterations, bool(fwd.converged)),
                    inverse_norm=Estimate(inv.value, inv.iterations, bool(inv.converged)),
                    has_factors=bool(hf.value))

    # error_bounds.hpp
    def loose_bounds(self, rn, bn, kappa):
        lo, hi = C.c_double(), C.c_double()
        st = self._f("loose_bounds")(C.c_double(rn), C.c_double(bn), C.c_double(kappa),
                                     C.byref(lo), C.byref(hi))
        if st:
            raise OracleError(st, "loose_bounds")
        return lo.value, hi.value

    def tight_bounds(self, rn, an, xn, kappa):
        lo, hi = C.c_double(), C.c_double()
        st = self._f("tight_bounds")(C.c_double(rn), C.c_double(an), C.c_double(xn),
                                     C.c_double(kappa), C.byref(lo), C.byref(hi))
        if st:
            raise OracleError(st, "tight_bounds")
        return lo.value, hi.value

    def propagate_bound(self, e):
        out = C.c_double()
        st = self._f("propagate_bound")(C.c_double(e), C.byref(out))
        if st:
            raise OracleError(st, "propagate_bound")
        return out.value

    def singularity_bound(self, kappa, eps=2.0 ** -53):
        out = C.c_double()
        st = self._f("singularity_bound")(C.c_double(kappa), C.c_double(eps), C.byref(out))
        if st:
            raise OracleError(st, "singularity_bound")
        return out.value

    def verify_solution(self, a, xhat, b, threshold=1e-7, kappa=None, a_norm=None,
                        eps_mach=2.0 ** -53, adam=None, restarts=3, pivot_tol=1e-14) -> dict:
        nr, nc, rp, ci, va = _csr(a)
        xhat = np.ascontiguousarray(xhat, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        o = VerifyOpts()
        o.threshold = threshold
        o.has_kappa, o.kappa = (1, kappa) if kappa is not None else (0, 0.0)
        o.has_a_norm, o.a_norm = (1, a_norm) if a_norm is not None else (0, 0.0)
        o.eps_mach = eps_mach
        o.adam = _cfg(adam) if adam is not None else AdamCfg(0.05, 0.9, 0.999, 1e-8, 2000, 1,
                                                              1e-12, 100)
        o.restarts, o.pivot_tol = restarts, pivot_tol
        rep = BoundsRep()
        st = self._f("verify_solution")(C.c_int64(nr), rp.ctypes.data_as(_i64p),
                                        ci.ctypes.data_as(_i32p), _d(va), _d(xhat), _d(b),
                                        C.byref(o), C.byref(rep))
        if st:
            raise OracleError(st, "verify_solution")
        return {k: getattr(rep, k) for k, _ in BoundsRep._fields_}

    # bench.py reference arm (ref backend only)
    def time_iterations(self, a, cfg, nthreads: int, iters: int):
        """Steady-state summed iterations/s of `nthreads` concurrent reference runs."""
        keep, args = self._csr_args(a)
        c = _cfg(cfg)
        rate, n, span = C.c_double(), C.c_uint64(), C.c_double()
        self._f("time_iterations")(*args, C.byref(c), C.c_int32(nthreads), C.c_uint64(iters),
                                   C.byref(rate), C.byref(n), C.byref(span))
        return rate.value, n.value, span.value

    def throughput_explicit(self, a, cfg, nthreads: int):
        keep, args = self._csr_args(a)
        c = _cfg(cfg)
        secs, its = C.c_double(), C.c_uint64()
        self._f("throughput_explicit")(*args, C.byref(c), C.c_int32(nthreads), C.byref(secs),
                                       C.byref(its))
        return secs.value, its.value
