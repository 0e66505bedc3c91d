"""Batched ensemble (config 5 shape) on the device vs per-member oracle runs."""
import numpy as np
import pytest

import matrices as M
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import batch, configs

pytestmark = pytest.mark.gpu


def _members(port):
    return [M.random_sparse(port, 77, 0.1, 3), configs.ensemble_member(0, 1, n=1000, bw=64),
            M.row_scaled(M.laplacian2d(20), port, 2), configs.ensemble_member(1, 1, n=513, bw=40),
            ck.SparseMatrix.identity(256)]


def test_pack_layout(port):
    mem = _members(port)
    a, seg_n = batch.pack_block_diagonal(mem)
    assert list(seg_n) == [m.nrows for m in mem]
    assert a.nrows == sum(-(-m.nrows // 256) * 256 for m in mem)
    x = np.concatenate([np.r_[port.random_unit_vectors(i, m.ncols)[0], np.zeros(-(-m.nrows // 256) * 256 - m.nrows)]
                        for i, m in enumerate(mem)])
    y = ck.matvec(a, x)
    off = 0
    for i, m in enumerate(mem):
        want = port.matvec(m, port.random_unit_vectors(i, m.ncols)[0])
        assert np.array_equal(y[off:off + m.nrows], want)
        off += -(-m.nrows // 256) * 256


def test_estimate_norm_batch_matches_members(port):
    mem = _members(port)
    cfg = M.cfg(alpha=1e-2, max_iter=400, patience=400)
    seeds = batch.member_seeds(len(mem))
    got = batch.estimate_norm_batch(mem, cfg, restarts=3, seeds=seeds)
    for m, g, sd in zip(mem, got, seeds):
        c = M.cfg(alpha=1e-2, max_iter=400, patience=400, seed=sd)
        o = port.estimate_norm_explicit(m, c, 3)
        alone = ck.estimate_norm(ck.ExplicitOracle(m), c, 3)
        assert g.iterations == o.iterations and g.converged == o.converged
        assert g.value == pytest.approx(o.value, rel=1e-9)
        assert g.value == pytest.approx(alone.value, rel=1e-12)


def test_batch_with_default_patience_and_zero_member(port):
    mem = [M.random_sparse(port, 30, 0.2, 5), ck.SparseMatrix.from_triplets(40, 40, []),
           M.diag_matrix([3.0, 1.0, 1e-3])]
    cfg = M.cfg()
    got = batch.estimate_norm_batch(mem, cfg, restarts=2, seeds=[7, 8, 9])
    for m, g, sd in zip(mem, got, [7, 8, 9]):
        o = port.estimate_norm_explicit(m, M.cfg(seed=sd), 2)
        assert g.iterations == o.iterations and g.converged == o.converged
        assert g.value == pytest.approx(o.value, rel=1e-9, abs=0.0)
    assert got[1].value == 0.0 and not got[1].converged


def test_batch_session_witnesses(port):
    mem = _members(port)[:3]
    packed = batch.pack_block_diagonal(mem)
    cfg = M.cfg(alpha=1e-2, max_iter=200, patience=200)
    seeds = [11 + k for k in range(len(mem) * 2)]
    s = batch.BatchSession(packed, cfg, seeds)
    assert s.run()
    for g, m in enumerate(mem):
        for c in range(2):
            e = s.member_result(g, c)
            o = port.projected_adam_explicit(m, M.cfg(alpha=1e-2, max_iter=200, patience=200,
                                                      seed=seeds[g * 2 + c]))
            assert e.value == pytest.approx(o.value, rel=1e-9)
            assert np.linalg.norm(m.to_dense() @ e.witness) == pytest.approx(e.value, rel=1e-12)


# ---------------------------------------------------------- sigma_min side
def _inv_members(port):
    return [M.random_sparse(port, 60, 0.2, 4), configs.ensemble_member(0, 1, n=1000, bw=64),
            M.row_scaled(M.laplacian2d(16), port, 2), configs.ensemble_member(1, 1, n=513, bw=40),
            M.diag_matrix([3.0, 1.0, 1e-3])]


def test_inverse_batch_matches_members(port):
    # one CTA per member: every member's run is the single-member run
    mem = _inv_members(port)
    facs = batch.lu_factorize_many(mem, 1e-14, threads=4)
    cfg = M.cfg(alpha=1e-2, max_iter=300, patience=300)
    seeds = batch.member_seeds(len(mem), 5)
    got = batch.inv_estimate_norm_batch(facs, cfg, restarts=3, seeds=seeds)
    for m, f, g, sd in zip(mem, facs, got, seeds):
        c = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=sd)
        alone = ck.estimate_norm(ck.InverseOracle(f), c, 3)
        # the batch sweeps 3 restart columns per member by substitution; a member alone
        # runs its restarts one CTA each, on the dense-block sweeps where the band is
        # narrow (ck_lu_dense.cuh): same solves to rounding
        assert g.value == pytest.approx(alone.value, rel=1e-11) and g.iterations == alone.iterations
        o = port.estimate_norm_inverse(port.lu_factorize(m, 1e-14), c, 3)
        assert g.iterations == o.iterations and g.converged == o.converged
        assert g.value == pytest.approx(o.value, rel=1e-9)


def test_inverse_batch_session_witnesses(port):
    mem = _inv_members(port)[:3]
    facs = batch.lu_factorize_many(mem, 1e-14, threads=1)
    cfg = M.cfg(alpha=1e-2, max_iter=150, patience=150)
    seeds = [21 + k for k in range(len(mem) * 2)]
    s = batch.InverseBatchSession(facs, cfg, seeds)
    assert s.run()
    for g, (m, f) in enumerate(zip(mem, facs)):
        for c in range(2):
            e = s.member_result(g, c)
            alone = ck.projected_adam(ck.InverseOracle(f), M.cfg(alpha=1e-2, max_iter=150,
                                                                  patience=150, seed=seeds[g * 2 + c]))
            # alone: one CTA per run on the dense-block sweeps (narrow bands); the
            # session sweeps 2 columns per member by substitution -- same solves to rounding
            assert e.value == pytest.approx(alone.value, rel=1e-11)
            assert np.linalg.norm(e.witness - alone.witness) <= 1e-9
            assert np.linalg.norm(f.solve(e.witness)) == pytest.approx(e.value, rel=1e-12)


def test_cond2_batch_matches_cond2(port):
    # bench.hpp:435 per-matrix cond2 with member seeds; a singular member -> inf
    dup = ck.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (0, 1, 2.0), (1, 0, 1.0), (1, 1, 2.0),
                                               (2, 2, 5.0)])
    mem = _inv_members(port)[:4] + [dup]
    cfg = M.cfg(alpha=1e-2, max_iter=300, patience=300)
    seeds = batch.member_seeds(len(mem), 3)
    got = batch.cond2_batch(mem, cfg, restarts=2, seeds=seeds, wave=2, threads=2)
    for m, r, sd in zip(mem[:4], got, seeds):
        c = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=sd)
        want = ck.cond2(m, c, restarts=2)
        assert r.kappa == pytest.approx(want.kappa, rel=1e-11)  # substitution vs dense-block sweeps
        o = port.cond2(m, c, restarts=2)
        assert r.kappa == pytest.approx(o["kappa"], rel=1e-9)
    assert got[4].kappa == float("inf")


def test_auto_wave_fills_the_device(port):
    """Default ensemble waves: one member per SM, within device memory."""
    mem = _inv_members(port)[:3]
    w = batch.auto_wave(mem)
    assert 3 <= w <= 1024
    got = batch.cond2_batch(mem, M.cfg(alpha=1e-2, max_iter=100, patience=100), restarts=2)
    want = batch.cond2_batch(mem, M.cfg(alpha=1e-2, max_iter=100, patience=100), restarts=2, wave=1)
    for g, h in zip(got, want):
        assert g.kappa == h.kappa


def test_window_sweeps_match_gathers_bitwise(port, monkeypatch):
    """Banded ensembles gather x~ / y' from a sliding shared-memory window (every
    column within one 256-row tile of its row); same operands, same order: the
    results are those of the global-memory gathers, bit for bit. A member with a
    far entry switches the whole batch to the gathers."""
    mem = [configs.ensemble_member(i, 1, n=n, bw=bw) for i, (n, bw) in
           enumerate([(3000, 200), (1500, 255), (700, 30), (2049, 128)])]
    cfg = M.cfg(alpha=1e-2, max_iter=150, patience=150)
    seeds = batch.member_seeds(len(mem))
    for restarts in (1, 2, 3, 4):
        win = batch.estimate_norm_batch(mem, cfg, restarts=restarts, seeds=seeds)
        monkeypatch.setenv("CK_NO_WINDOW", "1")
        ref = batch.estimate_norm_batch(mem, cfg, restarts=restarts, seeds=seeds)
        monkeypatch.delenv("CK_NO_WINDOW")
        for w, r in zip(win, ref):
            assert w.value == r.value and w.iterations == r.iterations
            assert np.array_equal(w.witness, r.witness)
    # reach > 1: entry (0, 900) in the first member
    far = mem[0]
    rp, ci, va = far.row_offsets.copy(), list(far.col_indices), list(far.values)
    trip = [(i, ci[k], va[k]) for i in range(far.nrows) for k in range(rp[i], rp[i + 1])]
    trip.append((0, 900, 0.5))
    far2 = ck.SparseMatrix.from_triplets(far.nrows, far.ncols, trip)
    got = batch.estimate_norm_batch([far2, mem[1]], cfg, restarts=2, seeds=seeds[:2])
    alone = ck.estimate_norm(ck.ExplicitOracle(far2), M.cfg(alpha=1e-2, max_iter=150, patience=150, seed=seeds[0]), 2)
    assert got[0].value == pytest.approx(alone.value, rel=1e-12)


def test_restart_group_query(port):
    """ck_restart_group: the grouping estimate_norm / estimate_norm_batch use (restarts are
    independent runs, condest.hpp:301-312; grouped for throughput only)."""
    import ctypes
    from paper_2409_11515_b200 import _lib

    def group(a, restarts, is_batch):
        g = ctypes.c_int32(0)
        _lib.check(_lib.load().ck_restart_group(a.device().handle, restarts, is_batch, ctypes.byref(g)),
                   "ck_restart_group")
        return g.value

    small = M.laplacian2d(16)
    assert group(small, 3, 0) == 4 and group(small, 4, 1) == 4  # below 2^24 nonzeros: 4 columns
