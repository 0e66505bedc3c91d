"""sigma_min path on the device vs the oracle: band LU (lu.hpp), triangular
solves, Projected Adam on A^-1 (InverseOracle), cond2 and verify_solution."""
import math

import numpy as np
import pytest

import matrices as M
import paper_2409_11515_b200 as ck

pytestmark = pytest.mark.gpu


def assert_same_factors(f, rf, a=None):
    """Device LUFactors (CSR export, lu.hpp:42-47 shape) == the oracle's, bit for bit."""
    e = rf.export()
    l, u, perm = f.export_csr()
    assert np.array_equal(perm, e["row_perm"])
    for mine, (rp, ci, va) in ((l, e["l"]), (u, e["u"])):
        assert np.array_equal(mine.row_offsets, rp)
        assert np.array_equal(mine.col_indices, ci)
        assert np.array_equal(mine.values.view(np.uint64), va.view(np.uint64))
    assert f.pivot_min == rf.pivot_min
    if a is not None and a.nrows <= 400:
        d = a.to_dense()
        L = l.to_dense() + np.eye(a.nrows)
        assert np.linalg.norm(d[perm] - L @ u.to_dense()) <= 1e-13 * np.linalg.norm(d)
        assert np.abs(l.values).max(initial=0.0) <= 1.0


@pytest.mark.parametrize("n,seed", [(5, 8), (20, 15), (50, 29), (50, 36), (100, 3)])
def test_factors_match_reference_bitwise(port, n, seed):
    # test_lu.cpp:54-70 fixtures; same pivots and unfused arithmetic -> same factors
    a = M.random_sparse(port, n, 0.3, seed)
    assert_same_factors(ck.lu_factorize(a, 1e-12), port.lu_factorize(a, 1e-12), a)


def test_long_band_factors_match_reference_bitwise(port):
    # n >> kl: fill carried across many 32-column panels (dgbtf2's running ju)
    from paper_2409_11515_b200 import configs
    a = configs.ensemble_member(3, 1, n=1500, bw=200)
    f = ck.lu_factorize(a, 1e-14)
    rf = port.lu_factorize(a, 1e-14)
    assert_same_factors(f, rf)
    b = port.random_unit_vectors(5, a.nrows)[0]
    assert np.linalg.norm(f.solve(b) - port.lu_solve(rf, b)) <= 1e-12 * np.linalg.norm(port.lu_solve(rf, b))


def test_identity_and_permutation():
    # test_lu.cpp:28-52
    f = ck.lu_factorize(ck.SparseMatrix.identity(4))
    assert f.pivot_min == 1.0
    assert np.array_equal(f.solve([1.0, 2.0, 3.0, 4.0]), [1.0, 2.0, 3.0, 4.0])
    a = ck.SparseMatrix.from_triplets(2, 2, [(0, 1, 1.0), (1, 0, 1.0)])
    f = ck.lu_factorize(a)
    assert f.pivot_min == 1.0
    assert np.array_equal(f.solve([1.0, 2.0]), [2.0, 1.0])
    assert np.array_equal(f.transpose_solve([3.0, 4.0]), [4.0, 3.0])
    f = ck.lu_factorize(M.diag_matrix([5.0, 3.0, 8.0]))
    assert f.pivot_min == 3.0


def _banded(n, bw, seed):
    rng = np.random.default_rng(seed)
    r, c, v = [], [], []
    for i in range(n):
        for j in range(max(0, i - bw), min(n, i + bw + 1)):
            if i == j or rng.random() < 0.3:
                r.append(i)
                c.append(j)
                v.append(rng.standard_normal() * (3.0 if i == j else 1.0))
    return ck.SparseMatrix.from_coo(n, n, r, c, v)


@pytest.mark.parametrize("kind", ["random40", "laplacian24", "banded700", "rowscaled33"])
def test_solves_match_reference(port, kind):
    a = {"random40": lambda: M.random_sparse(port, 40, 0.2, 4),
         "laplacian24": lambda: M.laplacian2d(24),
         "banded700": lambda: _banded(700, 45, 2),
         "rowscaled33": lambda: M.row_scaled(M.laplacian2d(33), port, 1)}[kind]()
    f = ck.lu_factorize(a, 1e-14)
    rf = port.lu_factorize(a, 1e-14)
    d = a.to_dense()
    for seed in (1, 2):
        b = port.random_unit_vectors(seed, a.nrows)[0]
        x, xr = f.solve(b), port.lu_solve(rf, b)
        assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)
        t, tr = f.transpose_solve(b), port.lu_transpose_solve(rf, b)
        assert np.linalg.norm(t - tr) <= 1e-12 * np.linalg.norm(tr)
        assert np.linalg.norm(d @ x - b) <= 1e-12 * np.linalg.norm(d) * np.linalg.norm(x)


def test_singular_factorisations():
    dup = ck.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (0, 1, 2.0), (1, 0, 1.0), (1, 1, 2.0),
                                               (2, 2, 5.0)])
    with pytest.raises(ck.NumericallySingular) as e:
        ck.lu_factorize(dup, 1e-14)
    assert e.value.column == 1
    empty = ck.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 0, 1.0)])
    with pytest.raises(ck.StructurallySingular) as e:
        ck.lu_factorize(empty, 1e-14)
    assert e.value.column == 2
    r = ck.cond2(dup)
    assert math.isinf(r.kappa) and math.isinf(r.inverse_norm.value)
    assert r.operator_norm.value > 0 and r.factors is None
    r = ck.cond2(ck.SparseMatrix.from_triplets(3, 3, []))
    assert math.isinf(r.kappa) and r.operator_norm.value == 0.0


def test_inverse_loss_grad(port):
    a = M.random_sparse(port, 20, 0.3, 7)
    f, rf = ck.lu_factorize(a), port.lu_factorize(a)
    ox = ck.InverseOracle(f)
    for x in port.random_unit_vectors(13, 20, 4):
        assert ox.loss(x) == pytest.approx(port.loss_inverse(rf, x), rel=1e-12, abs=1e-14)
        assert np.allclose(ox.grad(x), port.grad_inverse(rf, x), rtol=1e-11, atol=1e-14)


def test_inverse_known_norm():
    # test_condest.cpp:150-160
    f = ck.lu_factorize(M.diag_matrix([3.0, 1.0, 1e-3]))
    e = ck.inv_norm2(f)
    assert e.converged and e.value == pytest.approx(1e3, rel=1e-9)


@pytest.mark.parametrize("seed", [1, 2])
def test_inverse_projected_adam_vs_oracle(port, seed):
    a = M.row_scaled(M.laplacian2d(16), port, seed)
    c = M.cfg(alpha=1e-2, max_iter=2000, patience=2000, seed=seed)
    f, rf = ck.lu_factorize(a, 1e-14), port.lu_factorize(a, 1e-14)
    g = ck.projected_adam(ck.InverseOracle(f), c)
    o = port.projected_adam_inverse(rf, c)
    assert g.iterations == o.iterations and g.converged == o.converged
    assert g.value == pytest.approx(o.value, rel=1e-3)
    assert np.linalg.norm(port.lu_solve(rf, g.witness)) == pytest.approx(g.value, rel=1e-11)


def test_inverse_default_config_vs_oracle(port):
    a = M.random_sparse(port, 30, 0.2, 9)
    f, rf = ck.lu_factorize(a), port.lu_factorize(a)
    c = M.cfg(seed=4)
    g = ck.projected_adam(ck.InverseOracle(f), c)
    o = port.projected_adam_inverse(rf, c)
    assert g.iterations == o.iterations and g.converged == o.converged
    assert g.value == pytest.approx(o.value, rel=1e-9)
    e = ck.estimate_norm(ck.InverseOracle(f), c, 3)
    eo = port.estimate_norm_inverse(rf, c, 3)
    assert e.value == pytest.approx(eo.value, rel=1e-9)


def test_inverse_trajectory_invariants():
    # acceptance.cpp:319-352 for the inverse oracle
    a, _ = M.svd_constructed(30, M.geometric_sigmas(30, 2.0, 1e6), 44)
    f = ck.lu_factorize(a, 1e-14)
    prev_t, prev_min, calls = 0, math.inf, 0

    def obs(st, info):
        nonlocal prev_t, prev_min, calls
        calls += 1
        assert abs(np.linalg.norm(st.x) - 1.0) <= 1e-14
        assert abs(info.x_dot_delta) <= 1e-13 * info.delta_norm + 1e-300
        assert st.loss_min <= prev_min and st.t == prev_t + 1
        prev_t, prev_min = st.t, st.loss_min

    c = M.cfg(seed=13)
    e = ck.projected_adam(ck.InverseOracle(f), c, obs)
    again = ck.projected_adam(ck.InverseOracle(f), c)
    assert calls > 0 and e.value == again.value and np.array_equal(e.witness, again.witness)


@pytest.mark.parametrize("case", ["random30", "diag", "constructed1e8", "config1_shape"])
def test_cond2_vs_oracle(port, case):
    # test_condest.cpp:274-301 and the BASELINE config-1 recipe (on a 24x24 grid)
    if case == "random30":
        a, c, tol = M.random_sparse(port, 30, 0.3, 53), M.cfg(), 1e-9
    elif case == "diag":
        a, c, tol = M.diag_matrix([10.0, 2.0, 1.0]), M.cfg(), 1e-12
    elif case == "constructed1e8":
        a, c, tol = M.svd_constructed(40, M.geometric_sigmas(40, 1.0, 1e8), 77)[0], M.cfg(), 1e-3
    else:
        a = M.row_scaled(M.laplacian2d(24), port, 1)
        c, tol = M.cfg(alpha=1e-2, max_iter=2000, patience=2000), 1e-3
    r = ck.cond2(a, c)
    o = port.cond2(a, c)
    assert r.kappa == pytest.approx(o["kappa"], rel=tol)
    assert r.operator_norm.value == pytest.approx(o["operator_norm"].value, rel=tol)
    assert r.inverse_norm.value == pytest.approx(o["inverse_norm"].value, rel=tol)
    assert r.factors is not None


def test_cond2_against_dense_svd():
    a, d = M.svd_constructed(40, M.geometric_sigmas(40, 1.0, 1e8), 77)
    s = np.linalg.svd(d, compute_uv=False)
    r = ck.cond2(a)
    assert r.kappa == pytest.approx(s[0] / s[-1], rel=1e-3)
    assert r.operator_norm.converged and r.inverse_norm.converged


def test_verify_solution_vs_oracle(port):
    a = M.random_sparse(port, 40, 0.2, 3)
    x = port.uniform_in(70, 40, -1.0, 1.0)
    b = port.matvec(a, x)
    xh = x + 1e-6 * port.random_unit_vectors(4, 40)[0]
    rep = ck.verify_solution(a, xh, b)
    ro = port.verify_solution(a, xh, b)
    assert rep.residual_norm == pytest.approx(ro["residual_norm"], rel=1e-13)
    assert rep.kappa == pytest.approx(ro["kappa"], rel=1e-9)
    assert rep.loose_upper == pytest.approx(ro["loose_upper"], rel=1e-9)
    assert rep.verdict.value == ro["verdict"]
    rep = ck.verify_solution(a, xh, b, ck.VerifyOptions(kappa=50.0, a_norm=3.0))
    ro = port.verify_solution(a, xh, b, kappa=50.0, a_norm=3.0)
    for k in ("residual_norm", "b_norm", "xhat_norm", "loose_lower", "loose_upper", "tight_lower",
              "tight_upper", "true_error_cap", "singularity_cap"):
        assert getattr(rep, k) == pytest.approx(ro[k], rel=1e-13), k
    assert rep.kappa_supplied and len(rep.to_kv()) == 15
    with pytest.raises(ck.ZeroSolution):
        ck.verify_solution(a, np.zeros(40), b)
    with pytest.raises(ck.ZeroRHS):
        ck.verify_solution(a, xh, np.zeros(40))


def test_inverse_restarts_are_separate_runs(port):
    """estimate_norm on the InverseOracle runs every restart on its own CTA
    (batch members sharing the factors): the best restart is bit-identical to
    the separately seeded run (condest.hpp:301-312)."""
    a = M.row_scaled(M.laplacian2d(12), port, 3)
    f = ck.lu_factorize(a, 1e-14)
    c = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=11)
    comb = ck.estimate_norm(ck.InverseOracle(f), c, 4)
    best = None
    for r in range(4):
        cr = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=11 if r == 0 else ck.mix_seed(11, r))
        e = ck.projected_adam(ck.InverseOracle(f), cr)
        if best is None or e.value > best.value:
            best = e
    assert comb.value == best.value and comb.iterations == best.iterations
    assert np.array_equal(comb.witness, best.witness)


@pytest.mark.parametrize("cl", ["2", "8"])
def test_cluster_sweeps_match_single_cta_and_oracle(port, monkeypatch, cl):
    """The cluster split of the band sweeps (helpers stream the tail / dot
    coefficients, the leader keeps heads and the ring) agrees with the
    single-CTA sweeps and with the oracle."""
    a = M.row_scaled(M.laplacian2d(24), port, 5)
    f, rf = ck.lu_factorize(a, 1e-14), port.lu_factorize(a, 1e-14)
    c = M.cfg(alpha=1e-2, max_iter=400, patience=400, seed=9)
    monkeypatch.setenv("CK_LU_CLUSTER", "1")
    one = ck.projected_adam(ck.InverseOracle(f), c)
    monkeypatch.setenv("CK_LU_CLUSTER", cl)
    clu = ck.projected_adam(ck.InverseOracle(f), c)
    o = port.projected_adam_inverse(rf, c)
    assert clu.iterations == one.iterations == o.iterations
    assert clu.value == pytest.approx(one.value, rel=1e-12)
    assert clu.value == pytest.approx(o.value, rel=1e-9)
    assert np.linalg.norm(port.lu_solve(rf, clu.witness)) == pytest.approx(clu.value, rel=1e-11)


def test_cluster_sweeps_several_columns(port, monkeypatch):
    """Restart columns (R = 3) through the cluster split: every column agrees
    with the single-CTA sweep."""
    from paper_2409_11515_b200 import inverse
    a = M.row_scaled(M.laplacian2d(20), port, 7)
    f = ck.lu_factorize(a, 1e-14)
    c = M.cfg(alpha=1e-2, max_iter=200, patience=200, seed=4)
    res = {}
    for cl in ("1", "8"):
        monkeypatch.setenv("CK_LU_CLUSTER", cl)
        s = inverse.InverseSession(ck.InverseOracle(f), c, [4, 5, 6])
        assert s.run()
        res[cl] = [s.result(k) for k in range(3)]
    for e1, e8 in zip(res["1"], res["8"]):
        assert e8.iterations == e1.iterations
        assert e8.value == pytest.approx(e1.value, rel=1e-12)


@pytest.mark.parametrize("kind", ["random40", "laplacian24", "banded700", "rowscaled64", "odd1000", "tiny3",
                                  "limit190"])
def test_dense_block_sweeps_match_substitution(port, kind):
    """Narrow bands: the InverseOracle loop sweeps with the inverted 32 x 32 head
    triangles (ck_lu_dense.cuh). Same solves as lu_solve / lu_transpose_solve
    (lu.hpp:180-227): within 1e-10 of the oracle (observed ~1e-14), growth-guarded."""
    from paper_2409_11515_b200 import configs
    a = {"random40": lambda: M.random_sparse(port, 40, 0.2, 4),
         "laplacian24": lambda: M.laplacian2d(24),
         "banded700": lambda: _banded(700, 45, 2),
         "rowscaled64": lambda: M.row_scaled(M.laplacian2d(64), port, 1),
         "odd1000": lambda: _banded(1003, 70, 5),
         "limit190": lambda: _banded(900, 95, 9),  # kl + ku = 190: the widest band of the dense path
         "tiny3": lambda: M.diag_matrix([5.0, 3.0, 8.0])}[kind]()
    f = ck.lu_factorize(a, 1e-14)
    rf = port.lu_factorize(a, 1e-14)
    ok, growth = f.dense_info()
    assert ok and 1.0 <= growth <= 1e4
    for k in range(3):
        b = port.random_unit_vectors(11 + k, a.nrows)[0]
        for tr in (False, True):
            want = port.lu_transpose_solve(rf, b) if tr else port.lu_solve(rf, b)
            got = f.dense_solve(b, transpose=tr)
            assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
            exact = f.transpose_solve(b) if tr else f.solve(b)
            assert np.linalg.norm(got - exact) <= 1e-11 * np.linalg.norm(exact)


def test_dense_sweeps_guard_and_loop(port, monkeypatch):
    """Wide bands and ill-conditioned heads keep the substitution sweeps; on narrow
    bands the loop's sigma_min agrees with the substitution loop and the oracle."""
    from paper_2409_11515_b200 import configs
    wide = configs.ensemble_member(3, 1, n=1500, bw=150)  # kl + ku ~ 300 > 192
    assert not ck.lu_factorize(wide, 1e-14).dense_info()[0]
    ill = configs.ensemble_member(0, 1, n=600, bw=20)  # column scales 10^U(-8, 8)
    fi = ck.lu_factorize(ill, 1e-14)
    ok, growth = fi.dense_info()
    assert ok == (growth <= 1e4)
    a = M.row_scaled(M.laplacian2d(40), port, 3)
    cfg = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=5)
    dense = ck.inv_norm2(ck.lu_factorize(a, 1e-14), cfg)
    monkeypatch.setenv("CK_LU_DENSE", "0")
    subst = ck.inv_norm2(ck.lu_factorize(a, 1e-14), cfg)
    monkeypatch.delenv("CK_LU_DENSE")
    want = port.projected_adam_inverse(port.lu_factorize(a, 1e-14), cfg)
    assert dense.iterations == subst.iterations == want.iterations
    assert dense.value == pytest.approx(subst.value, rel=1e-9)
    assert dense.value == pytest.approx(want.value, rel=1e-9)
