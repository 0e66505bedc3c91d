"""Host logic of the row-block partition at world size 2 over gloo (CPU):
each rank builds its extended operator, exchanges halo needs with
all_gather_object, then runs y = A x and z = A^T y with real send/recv of
the halo values over the lists -- bit-identical to the global products
(oracle arithmetic: stored-order sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(me, side, values_own_ext, world):
    """Send the listed own entries, receive the halo entries (global order)."""
    L = me.lists
    so, si, ro, ri = L[side + "s_off"], L[side + "s_idx"], L[side + "r_off"], L[side + "r_idx"]
    reqs, recv = [], {}
    for q in range(world):
        if q == me.rank:
            continue
        if so[q + 1] > so[q]:
            reqs.append(tdist.isend(torch.from_numpy(values_own_ext[si[so[q]:so[q + 1]]].copy()), q))
        if ro[q + 1] > ro[q]:
            buf = torch.empty(int(ro[q + 1] - ro[q]), dtype=torch.float64)
            reqs.append(tdist.irecv(buf, q))
            recv[q] = buf
    for r in reqs:
        r.wait()
    for q, buf in recv.items():
        values_own_ext[ri[ro[q]:ro[q + 1]]] = buf.numpy()
    return values_own_ext


def _worker(rank, world, port, kind, out):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import pyoracle
        import matrices as M
        from paper_2409_11515_b200 import dist
        from paper_2409_11515_b200.sparse import SparseMatrix
        port_ = pyoracle.Oracle("port")
        a = {"lap": lambda: M.row_scaled(M.laplacian2d(36), port_, 1),
             "rand": lambda: M.random_sparse(port_, 400, 0.02, 7)}[kind]()

        def gather(obj):
            res = [None] * world
            tdist.all_gather_object(res, obj)
            return res

        me = dist.build_rank(a, world, rank, gather)
        ref = dist.build_partition(a, world)[rank]
        for k in ref.lists:  # every rank derives the same lists as the all-in-one build
            assert np.array_equal(me.lists[k], ref.lists[k]), k
        x = port_.random_unit_vectors(11, a.ncols)[0]
        C_ = SparseMatrix(me.ext_rows, me.ext_cols, me.rp, me.ci, me.va)
        xe = np.zeros(me.ext_cols)
        xe[me.own_offset():me.own_offset() + me.n_loc] = x[me.g0:me.g1]
        xe = _exchange(me, "x", xe, world)
        ye = port_.matvec(C_, xe)
        y_own = ye[me.own_offset():me.own_offset() + me.n_loc].copy()
        yfull = port_.matvec(a, x)
        ok_y = np.array_equal(y_own, yfull[me.g0:me.g1])
        ye[:] = 0.0
        ye[me.own_offset():me.own_offset() + me.n_loc] = y_own
        ye = _exchange(me, "y", ye, world)
        ze = port_.transpose_matvec(C_, ye)
        ok_z = np.array_equal(ze[me.own_offset():me.own_offset() + me.n_loc],
                              port_.transpose_matvec(a, yfull)[me.g0:me.g1])
        # per-rank partials merged in rank order: identical scalars on every rank
        part = torch.tensor([float(np.dot(y_own, y_own))], dtype=torch.float64)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        tdist.all_gather(parts, part)
        tot = sum(float(t) for t in parts)
        out[rank] = (ok_y, ok_z, tot)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("kind", ["lap", "rand"])
def test_two_rank_halo_exchange_gloo(kind):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), kind, out), nprocs=world, join=True)
    assert all(out[r][0] for r in range(world)), "y = A x"
    assert all(out[r][1] for r in range(world)), "z = A^T y"
    assert out[0][2] == out[1][2]


def test_partition_bounds_and_positions():
    import sys
    sys.path[:0] = [os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
    import pyoracle
    import matrices as M
    from paper_2409_11515_b200 import dist
    port_ = pyoracle.Oracle("port")
    a = M.random_sparse(port_, 300, 0.03, 2)
    for P in (1, 2, 4, 7):
        b = dist.partition_rows(a, P)
        assert b[0] == 0 and b[-1] == a.nrows and np.all(np.diff(b) > 0)
        parts = dist.build_partition(a, P)
        for p in parts:
            cols = p.ext_global[p.ext_global >= 0]
            assert np.all(np.diff(cols) > 0)  # extended order = global order
            assert p.tile0 * 256 >= (p.hx < p.g0).sum() and p.tile0 * 256 >= (p.hy < p.g0).sum()
            assert np.all(np.diff(p.rp) >= 0) and p.rp[-1] == p.ci.size
