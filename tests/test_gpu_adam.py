"""Projected Adam on the device vs the CPU oracle (condest.hpp:184-312)."""
import math

import numpy as np
import pytest

import matrices as M
import paper_2409_11515_b200 as ck

pytestmark = pytest.mark.gpu

TOL = 1e-3  # north_star: sigma within 1e-3 relative after the same iteration count


def _cmp(port, a, c, tol=1e-9):
    g = ck.norm2(a, c)
    o = port.projected_adam_explicit(a, c)
    assert g.iterations == o.iterations
    assert g.converged == o.converged
    assert g.value == pytest.approx(o.value, rel=tol)
    return g, o


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_config1_shape_sigma_max(port, seed):
    # BASELINE config 1 recipe at 32x32 (row-scaled Dirichlet Laplacian, alpha 1e-2, patience off)
    a = M.row_scaled(M.laplacian2d(32), port, seed)
    c = M.cfg(alpha=1e-2, max_iter=2000, patience=2000, seed=seed)
    g, o = _cmp(port, a, c, tol=TOL)
    assert abs(np.linalg.norm(g.witness) - 1.0) < 1e-14
    # the witness is the same direction (up to the rounding-driven trajectory)
    assert np.linalg.norm(a.to_dense() @ g.witness) == pytest.approx(g.value, rel=1e-12)


def test_early_iterations_track_oracle_closely(port):
    a = M.row_scaled(M.laplacian2d(16), port, 5)
    c = M.cfg(alpha=1e-2, max_iter=50, patience=50, seed=5)
    g, o = _cmp(port, a, c, tol=1e-12)
    assert np.allclose(g.witness, o.witness, rtol=0, atol=1e-12)


def test_default_config_with_patience(port):
    for s in (31, 32):
        a = M.random_sparse(port, 30, 0.2, s)
        _cmp(port, a, M.cfg(seed=2), tol=1e-9)


def test_known_norms():
    # test_condest.cpp:140-180
    e = ck.norm2(ck.SparseMatrix.identity(10))
    assert abs(e.value - 1.0) <= 1e-12 and e.converged and e.iterations < 2000
    assert abs(np.linalg.norm(e.witness) - 1.0) <= 1e-14
    e = ck.norm2(M.diag_matrix([3.0, 1.0, 1e-3]))
    assert e.converged and e.value == pytest.approx(3.0, rel=1e-9)
    z = ck.norm2(ck.SparseMatrix.from_triplets(4, 4, []))
    assert z.value == 0.0 and not z.converged


def test_constructed_spectrum():
    a, d = M.svd_constructed(40, M.geometric_sigmas(40, 1.0, 1e8), 5)
    est = ck.estimate_norm(ck.ExplicitOracle(a))
    smax = np.linalg.svd(d, compute_uv=False)[0]
    assert est.value <= smax * (1 + 1e-12)
    assert est.value == pytest.approx(smax, rel=1e-4)
    assert est.value == pytest.approx(np.linalg.norm(d @ est.witness), rel=1e-14)


def test_restarts_are_independent_columns(port):
    # estimate_norm == best of separately seeded runs, bit for bit (test_condest.cpp:250-265)
    a = M.random_sparse(port, 25, 0.25, 17)
    c = M.cfg(seed=7)
    comb = ck.estimate_norm(ck.ExplicitOracle(a), c, 3)
    best = None
    for r in range(3):
        cc = M.cfg(seed=7 if r == 0 else ck.mix_seed(7, r))
        e = ck.norm2(a, cc)
        if best is None or e.value > best.value:
            best = e
    assert comb.value == best.value
    assert np.array_equal(comb.witness, best.witness)
    o = port.estimate_norm_explicit(a, c, 3)
    assert comb.value == pytest.approx(o.value, rel=1e-9)


def test_five_restarts_span_two_sweeps(port):
    a = M.random_sparse(port, 40, 0.1, 4)
    c = M.cfg(seed=3)
    g = ck.estimate_norm(ck.ExplicitOracle(a), c, 5)
    o = port.estimate_norm_explicit(a, c, 5)
    assert g.value == pytest.approx(o.value, rel=1e-9)


def test_bitwise_determinism(port):
    a = M.random_sparse(port, 25, 0.25, 17)
    c = M.cfg(seed=42)
    e1, e2 = ck.norm2(a, c), ck.norm2(a, c)
    assert e1.value == e2.value and e1.iterations == e2.iterations
    assert np.array_equal(e1.witness, e2.witness)


def test_trajectory_invariants(port):
    # test_condest.cpp:182-220 through the observer
    for a, seed in [(M.random_sparse(port, 30, 0.2, 31), 2),
                    (M.svd_constructed(50, M.geometric_sigmas(50, 2.0, 1e6), 33)[0], 9)]:
        calls, prev_t, prev_min = 0, 0, math.inf

        def obs(st, info):
            nonlocal calls, prev_t, prev_min
            calls += 1
            assert abs(np.linalg.norm(st.x) - 1.0) <= 1e-14
            assert abs(info.x_dot_delta) <= 1e-13 * info.delta_norm
            assert st.loss_min <= prev_min
            assert st.t == prev_t + 1
            prev_t, prev_min = st.t, st.loss_min

        est = ck.projected_adam(ck.ExplicitOracle(a), M.cfg(seed=seed), obs)
        assert calls >= 1 and est.iterations == prev_t and est.converged


def test_observer_matches_plain_run(port):
    a = M.random_sparse(port, 30, 0.2, 8)
    c = M.cfg(seed=4)
    seen = []
    e1 = ck.projected_adam(ck.ExplicitOracle(a), c, lambda st, info: seen.append(info.loss))
    e2 = ck.norm2(a, c)
    assert e1.value == e2.value and e1.iterations == e2.iterations
    tr = port.projected_adam_explicit(a, c, trace=True).trace
    assert np.allclose(np.array(seen), tr[: len(seen)], rtol=1e-12, atol=1e-14)


def test_loss_and_grad_device(port):
    a = M.random_sparse(port, 20, 0.3, 7)
    ox = ck.ExplicitOracle(a)
    for x in port.random_unit_vectors(11, 20, 4):
        assert ox.loss(x) == pytest.approx(port.loss_explicit(a, x), rel=1e-14, abs=1e-15)
        assert np.allclose(ox.grad(x), port.grad_explicit(a, x), rtol=1e-13, atol=1e-15)
    z = ck.SparseMatrix.from_triplets(2, 2, [(0, 0, 1.0)])
    with pytest.raises(ck.DegenerateDirection):
        ck.loss_explicit(z, [0.0, 1.0])
    with pytest.raises(ck.DegenerateDirection):
        ck.grad_explicit(z, [0.0, 1.0])


def test_argument_validation():
    with pytest.raises(ValueError):
        ck.estimate_norm(ck.ExplicitOracle(ck.SparseMatrix.identity(3)), ck.AdamConfig(), 0)
    e = ck.norm2(ck.SparseMatrix.identity(3), M.cfg(max_iter=0))
    assert e.iterations == 0 and e.value == 0.0 and not e.converged


def test_degenerate_restarts_match_oracle(port):
    # a rank-1 operator: random starts are almost never degenerate, so force
    # one through a matrix with an empty column block and start vectors that
    # hit it only by restart; compare the full run against the oracle.
    a = ck.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0)])
    c = M.cfg(seed=5, max_iter=300)
    g = ck.norm2(a, c)
    o = port.projected_adam_explicit(a, c)
    assert g.iterations == o.iterations and g.converged == o.converged
    assert g.value == pytest.approx(o.value, rel=1e-12)


def test_rectangular(port):
    rng = np.random.default_rng(3)
    d = rng.standard_normal((30, 50)) * (rng.random((30, 50)) < 0.3)
    r, cidx = np.nonzero(d)
    a = ck.SparseMatrix.from_coo(30, 50, r, cidx, d[r, cidx])
    _cmp(port, a, M.cfg(seed=3), tol=1e-9)


def test_restart_grouping_is_invisible(port, monkeypatch):
    """Restart columns per sweep (CK_RESTART_GROUP) change nothing on a
    one-tile operator: every restart is the same run."""
    a = M.random_sparse(port, 40, 0.15, 21)
    c = M.cfg(seed=5)
    ref = ck.estimate_norm(ck.ExplicitOracle(a), c, 4)
    for g in ("1", "2", "3"):
        monkeypatch.setenv("CK_RESTART_GROUP", g)
        e = ck.estimate_norm(ck.ExplicitOracle(a), c, 4)
        assert e.value == ref.value and e.iterations == ref.iterations
        assert np.array_equal(e.witness, ref.witness)


def test_start_vector_prefetch_is_invisible():
    # ck_start_vector_prefetch (the first start vector drawn during the upload)
    # must give the same run bit for bit as drawing it inside the session; a
    # prefetch for another seed is ignored.
    from paper_2409_11515_b200 import _lib
    lap = M.laplacian2d(1024)  # n = 2^20: Session prefetches while A uploads
    c = M.cfg(alpha=1e-2, max_iter=40, patience=40, seed=9)

    def fresh():
        return ck.SparseMatrix(lap.nrows, lap.ncols, lap.row_offsets, lap.col_indices, lap.values)

    import ctypes as C
    lib = _lib.load()

    def stats():
        t, d = C.c_uint64(), C.c_uint64()
        _lib.check(lib.ck_start_vector_prefetch_stats(C.byref(t), C.byref(d)), "stats")
        return t.value, d.value

    t0, d0 = stats()
    e1 = ck.norm2(fresh(), c)  # prefetched
    assert stats() == (t0 + 1, d0)  # the session took the prefetched vector
    a2 = fresh()
    a2.device()
    e2 = ck.norm2(a2, c)  # drawn in the session
    assert stats() == (t0 + 1, d0)
    _lib.check(lib.ck_start_vector_prefetch(10, lap.ncols), "prefetch")
    e3 = ck.norm2(a2, c)  # stale slot (seed 10): dropped, drawn in the session
    assert stats() == (t0 + 1, d0 + 1)
    _lib.check(lib.ck_start_vector_prefetch(10, lap.ncols), "prefetch")
    _lib.check(lib.ck_start_vector_prefetch_cancel(), "cancel")
    assert stats() == (t0 + 1, d0 + 2)
    for e in (e2, e3):
        assert e.value == e1.value and e.iterations == e1.iterations
        assert np.array_equal(e.witness, e1.witness)
