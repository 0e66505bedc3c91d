"""Row-block partition of one operator across ranks.

Rank p owns the contiguous global rows/columns [g0, g1) -- nnz-balanced --
and runs the fused Projected-Adam kernels over its own block of an
*extended* local operator; halos of x~ and y' move between ranks every half
step and the per-rank reduction partials are all-gathered and merged in rank
order (ck_dist.cu). This module is the host side: the partition, the extended
operators, the halo lists and the session wrappers.

Extended index spaces (rows and columns alike), in increasing global order:
    [pad | left halo | own block, padded to whole 256-row tiles | right halo]
so every row of the extended operator keeps the reference's entry order and
the sparse products are bit-identical to one device.

Backends: ``nccl_id=None`` drives every rank in this process on one device
(lockstep, device copies for the collectives); otherwise one rank per
process over NCCL (``nccl_unique_id`` on rank 0, broadcast by the caller,
e.g. with ``torch.distributed.broadcast_object_list``).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .condest import AdamConfig, NormEstimate
from .sparse import SparseMatrix

TILE = 256


def partition_rows(a: SparseMatrix, nparts: int) -> np.ndarray:
    """Contiguous row ranges with about nnz/nparts entries each: bounds[p]..bounds[p+1]."""
    if a.nrows != a.ncols:
        raise ValueError("partition: square operators only")
    if not 1 <= nparts <= a.nrows:
        raise ValueError("partition: 1 <= nparts <= n")
    rp = a.row_offsets
    cuts = np.searchsorted(rp, np.arange(1, nparts) * (a.nnz / nparts), side="left")
    b = np.concatenate([[0], cuts, [a.nrows]]).astype(np.int64)
    for p in range(1, nparts + 1):  # every range non-empty
        b[p] = max(b[p], b[p - 1] + 1)
    for p in range(nparts - 1, -1, -1):
        b[p] = min(b[p], b[p + 1] - 1)
    return b


@dataclass
class Part:
    """Rank p's extended local operator and halo needs (global indices)."""
    rank: int
    n_global: int
    g0: int
    g1: int
    tile0: int
    tile1: int
    ext_rows: int
    ext_cols: int
    rp: np.ndarray
    ci: np.ndarray
    va: np.ndarray
    ext_global: np.ndarray   # extended column position -> global column (-1 padding)
    hx: np.ndarray           # global columns needed from other ranks (sorted)
    hy: np.ndarray           # global rows needed from other ranks (sorted)
    lists: dict = field(default_factory=dict, repr=False)

    @property
    def n_loc(self) -> int:
        return self.g1 - self.g0

    def own_offset(self) -> int:
        return self.tile0 * TILE

    def col_position(self, j: np.ndarray) -> np.ndarray:
        """Extended column positions of global columns j (own or halo)."""
        j = np.asarray(j, np.int64)
        out = np.empty(j.size, np.int64)
        own = (j >= self.g0) & (j < self.g1)
        out[own] = self.own_offset() + j[own] - self.g0
        left, right = self.hx[self.hx < self.g0], self.hx[self.hx >= self.g1]
        m = j < self.g0
        out[m] = self.own_offset() - left.size + np.searchsorted(left, j[m])
        m = j >= self.g1
        out[m] = self.tile1 * TILE + np.searchsorted(right, j[m])
        return out

    def row_position(self, i: np.ndarray) -> np.ndarray:
        """Extended row positions of global rows i (own or halo)."""
        i = np.asarray(i, np.int64)
        out = np.empty(i.size, np.int64)
        own = (i >= self.g0) & (i < self.g1)
        out[own] = self.own_offset() + i[own] - self.g0
        left, right = self.hy[self.hy < self.g0], self.hy[self.hy >= self.g1]
        m = i < self.g0
        out[m] = self.own_offset() - left.size + np.searchsorted(left, i[m])
        m = i >= self.g1
        out[m] = self.tile1 * TILE + np.searchsorted(right, i[m])
        return out


def _runs(starts: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """Concatenated index ranges [starts[k], starts[k] + lens[k])."""
    total = int(lens.sum())
    if total == 0:
        return np.zeros(0, np.int64)
    first = np.concatenate([[0], np.cumsum(lens)[:-1]])
    return np.repeat(starts - first, lens) + np.arange(total, dtype=np.int64)


def build_part(a: SparseMatrix, bounds: np.ndarray, p: int) -> Part:
    """Rank p's extended operator: own rows (complete) and the halo rows
    restricted to own columns, in increasing global order on both axes.
    One vectorised pass over the column indices finds the halo rows (rows
    with entries in own columns); their own-column entries are one
    contiguous run of each (sorted) row."""
    n = a.nrows
    g0, g1 = int(bounds[p]), int(bounds[p + 1])
    rp, ci, va = a.row_offsets, a.col_indices, a.values
    own_ci = ci[rp[g0]:rp[g1]].astype(np.int64)
    hx = np.unique(own_ci[(own_ci < g0) | (own_ci >= g1)])
    inside = (ci >= g0) & (ci < g1)
    before = ci < g0
    cin = np.concatenate([[0], np.cumsum(inside, dtype=np.int64)])
    cbe = np.concatenate([[0], np.cumsum(before, dtype=np.int64)])
    del inside, before
    cnt = cin[rp[1:]] - cin[rp[:-1]]  # own-column entries per row
    rows_hit = np.flatnonzero(cnt)
    hy = rows_hit[(rows_hit < g0) | (rows_hit >= g1)].astype(np.int64)
    nl = g1 - g0
    lx, ly = int((hx < g0).sum()), int((hy < g0).sum())
    tile0 = max(-(-lx // TILE), -(-ly // TILE))
    tile1 = tile0 + -(-nl // TILE)
    part = Part(p, n, g0, g1, tile0, tile1, tile1 * TILE + int((hy >= g1).sum()),
                tile1 * TILE + int((hx >= g1).sum()), None, None, None, None, hx, hy)
    lens = np.zeros(part.ext_rows, np.int64)
    lens[part.own_offset():part.own_offset() + nl] = np.diff(rp[g0:g1 + 1])
    hpos = part.row_position(hy)
    hlo = rp[hy] + (cbe[rp[hy + 1]] - cbe[rp[hy]])  # first own-column entry of each halo row
    hlen = cnt[hy]
    lens[hpos] = hlen
    out_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out_ci = np.empty(out_rp[-1], np.int64)
    out_va = np.empty(out_rp[-1])
    o0 = out_rp[part.own_offset()]
    seg = slice(rp[g0], rp[g1])
    out_ci[o0:o0 + (rp[g1] - rp[g0])] = part.col_position(own_ci)
    out_va[o0:o0 + (rp[g1] - rp[g0])] = va[seg]
    src = _runs(hlo, hlen)
    dst = _runs(out_rp[hpos], hlen)
    out_ci[dst] = part.col_position(ci[src])
    out_va[dst] = va[src]
    part.rp, part.ci, part.va = out_rp, out_ci.astype(np.int32), out_va
    eg = np.full(part.ext_cols, -1, np.int64)
    cols_all = np.concatenate([hx[hx < g0], np.arange(g0, g1, dtype=np.int64), hx[hx >= g1]])
    eg[part.col_position(cols_all)] = cols_all
    part.ext_global = eg
    return part


def halo_lists(parts_needs: Sequence[tuple], bounds: np.ndarray, me: Part) -> dict:
    """Send/receive lists of rank `me` from every rank's (hx, hy) needs.

    xs/ys: positions of own columns/rows rank q needs, in me's extended
    space; xr/yr: where rank q's values land in me's extended space. Within
    a (sender, receiver) pair both sides list the global indices ascending."""
    P = len(bounds) - 1
    out = {}
    for side, (need_idx, pos_fn) in {"x": (0, me.col_position), "y": (1, me.row_position)}.items():
        s_off, s_idx, r_off, r_idx = [0], [], [0], []
        mine = parts_needs[me.rank][need_idx]
        for q in range(P):
            if q == me.rank:
                s_off.append(s_off[-1])
                r_off.append(r_off[-1])
                continue
            theirs = parts_needs[q][need_idx]
            send = theirs[(theirs >= me.g0) & (theirs < me.g1)]
            recv = mine[(mine >= bounds[q]) & (mine < bounds[q + 1])]
            s_idx.append(pos_fn(send))
            r_idx.append(pos_fn(recv))
            s_off.append(s_off[-1] + send.size)
            r_off.append(r_off[-1] + recv.size)
        cat = lambda v: (np.concatenate(v) if v else np.zeros(0, np.int64)).astype(np.int32)  # noqa: E731
        out[side + "s_off"] = np.array(s_off, np.int64)
        out[side + "s_idx"] = cat(s_idx)
        out[side + "r_off"] = np.array(r_off, np.int64)
        out[side + "r_idx"] = cat(r_idx)
    return out


def build_partition(a: SparseMatrix, nparts: int) -> list[Part]:
    """Every rank's part and halo lists (in-process backend / tests)."""
    b = partition_rows(a, nparts)
    parts = [build_part(a, b, p) for p in range(nparts)]
    needs = [(p.hx, p.hy) for p in parts]
    for p in parts:
        p.lists = halo_lists(needs, b, p)
    return parts


def build_rank(a: SparseMatrix, nparts: int, rank: int, all_gather_object,
               bounds: Optional[np.ndarray] = None) -> Part:
    """This rank's part; the halo needs of all ranks are exchanged with
    `all_gather_object(obj) -> list` (e.g. torch.distributed's)."""
    b = partition_rows(a, nparts) if bounds is None else np.asarray(bounds, np.int64)
    me = build_part(a, b, rank)
    needs = all_gather_object((me.hx, me.hy))
    me.lists = halo_lists(needs, b, me)
    return me


# ------------------------------------------------------------------ sessions
class _PartC(C.Structure):
    _fields_ = [("n_global", C.c_int64), ("tile0", C.c_int64), ("tile1", C.c_int64),
                ("ext_rows", C.c_int64), ("ext_cols", C.c_int64),
                ("rp", C.c_void_p), ("ci", C.c_void_p), ("va", C.c_void_p),
                ("xs_off", C.c_void_p), ("xs_idx", C.c_void_p), ("xr_off", C.c_void_p),
                ("xr_idx", C.c_void_p), ("ys_off", C.c_void_p), ("ys_idx", C.c_void_p),
                ("yr_off", C.c_void_p), ("yr_idx", C.c_void_p), ("ext_global", C.c_void_p)]


def _as_c(p: Part, keep: list) -> _PartC:
    arrs = [np.ascontiguousarray(x) for x in
            (p.rp, p.ci, p.va, p.lists["xs_off"], p.lists["xs_idx"], p.lists["xr_off"],
             p.lists["xr_idx"], p.lists["ys_off"], p.lists["ys_idx"], p.lists["yr_off"],
             p.lists["yr_idx"], p.ext_global)]
    keep.extend(arrs)
    return _PartC(p.n_global, p.tile0, p.tile1, p.ext_rows, p.ext_cols,
                  *[x.ctypes.data for x in arrs])


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _lib.check(_lib.load().ck_dist_nccl_id(C.cast(buf, C.c_void_p)), "ck_dist_nccl_id")
    return bytes(buf)


class PartitionedSession:
    """Projected Adam over a row-block partition: `parts` are the ranks this
    process drives (all of them without nccl_id; exactly one with it)."""

    def __init__(self, parts: Sequence[Part], cfg: AdamConfig, seeds, nranks: Optional[int] = None,
                 nccl_id: Optional[bytes] = None):
        self.parts = list(parts)
        self.nranks = nranks or len(self.parts)
        seeds = np.ascontiguousarray([int(s) & 0xFFFFFFFFFFFFFFFF for s in seeds], np.uint64)
        self.ncols = seeds.size
        keep: list = []
        arr = (_PartC * len(self.parts))(*[_as_c(p, keep) for p in self.parts])
        lib = _lib.load()
        _lib.ensure_device()
        self._cfg = _lib.cfg_struct(cfg)
        self._id = None if nccl_id is None else (C.c_ubyte * 128).from_buffer_copy(nccl_id)
        idp = None if self._id is None else C.cast(self._id, C.c_void_p)
        h = C.c_void_p()
        _lib.check(lib.ck_dist_create(C.cast(arr, C.c_void_p), len(self.parts), self.parts[0].rank,
                                      self.nranks, idp, C.byref(self._cfg),
                                      seeds.ctypes.data_as(_lib.u64p),
                                      self.ncols, C.byref(h)), "ck_dist_create")
        self.handle = h
        self._fin = weakref.finalize(self, lib.ck_dist_free, h)

    def run(self, max_steps: int = 0) -> bool:
        fin = C.c_int32(0)
        _lib.check(_lib.load().ck_dist_run(self.handle, max_steps, C.byref(fin)), "ck_dist_run")
        return bool(fin.value)

    def time(self, steps: int) -> float:
        ms = C.c_double(0.0)
        _lib.check(_lib.load().ck_dist_time(self.handle, steps, C.byref(ms)), "ck_dist_time")
        return ms.value

    def info(self, part: int = 0) -> dict:
        """Device layout of part `part`'s extended local operator."""
        inf = _lib.MatrixInfo()
        _lib.check(_lib.load().ck_dist_part_info(self.handle, part, C.byref(inf)),
                   "ck_dist_part_info")
        return {k: getattr(inf, k) for k, _ in _lib.MatrixInfo._fields_}

    def result(self, col: int = 0, part: int = 0) -> NormEstimate:
        """Estimate of restart column `col`; witness = rank `part`'s own slice."""
        r = _lib.NormResult()
        p = self.parts[part]
        w = np.empty(p.ext_cols)
        _lib.check(_lib.load().ck_dist_result(self.handle, col, part, C.byref(r), _lib.dptr(w)),
                   "ck_dist_result")
        own = w[p.own_offset():p.own_offset() + p.n_loc]
        return NormEstimate(r.value, own, int(r.iterations), bool(r.converged))

    def free(self) -> None:
        self._fin()


def projected_adam_partitioned(a: SparseMatrix, nparts: int, cfg: Optional[AdamConfig] = None,
                               seeds: Optional[Sequence[int]] = None) -> list[NormEstimate]:
    """projected_adam (condest.hpp:184-297) of every seed over an in-process
    nparts-way row partition; witnesses assembled to global vectors."""
    cfg = cfg or AdamConfig()
    parts = build_partition(a, nparts)
    s = PartitionedSession(parts, cfg, seeds if seeds is not None else [cfg.seed])
    s.run()
    out = []
    for c in range(s.ncols):
        pieces = [s.result(c, p) for p in range(nparts)]
        w = np.concatenate([e.witness for e in pieces])
        out.append(NormEstimate(pieces[0].value, w, pieces[0].iterations, pieces[0].converged))
    s.free()
    return out
