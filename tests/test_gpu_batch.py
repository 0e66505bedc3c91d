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
