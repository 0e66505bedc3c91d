"""Pins the plain-C oracle (oracle/condkit_oracle.c) to the reference: against
the compiled reference itself (oracle/_ref, bit-for-bit) where it was built,
and against the reference tests' own known answers everywhere (CPU only)."""
import math

import numpy as np
import pytest

import matrices as M


def test_mt19937_64_known_answer(oracles):
    # The C++ standard fixes the 10000th output of a default-seeded mt19937_64.
    for o in oracles:
        assert int(o.mt_draws(5489, 10000)[-1]) == 9981545732273789042


def test_mix_seed_matches_reference(port, ref):
    for b, s in [(1, 0), (1, 1), (42, 0x1234), (2**63 + 5, 7)]:
        assert port.mix_seed(b, s) == ref.mix_seed(b, s)


def test_random_unit_vector_bitwise(port, ref):
    a = port.random_unit_vectors(3, 257, 4)
    b = ref.random_unit_vectors(3, 257, 4)
    assert np.array_equal(a, b)
    assert abs(port.two_norm(a[0]) - 1.0) < 1e-15


def test_two_norm_known_answers(oracles):
    # test_sparse.cpp:44-54
    for o in oracles:
        assert o.two_norm([3.0, 4.0]) == 5.0
        assert o.two_norm([]) == 0.0
        assert o.two_norm([3e300, 4e300]) == pytest.approx(5e300, rel=1e-15)
        assert o.two_norm(np.full(25, 1e300)) == pytest.approx(5e300, rel=1e-15)


def test_loss_grad_closed_forms(oracles):
    # test_condest.cpp:58-83
    a = M.diag_matrix([2.0, 1.0])
    s = 1.0 / math.sqrt(2.0)
    for o in oracles:
        assert o.loss_explicit(a, [s, s]) == pytest.approx(-0.5 * math.log(2.5), rel=1e-15)
        g = o.grad_explicit(a, [s, s])
        assert g[0] == pytest.approx(s * (1.0 - 4.0 / 2.5), rel=1e-14)
        assert g[1] == pytest.approx(s * (1.0 - 1.0 / 2.5), rel=1e-14)
        for x in ([1.0, 0.0], [0.0, 1.0]):
            assert np.all(np.abs(o.grad_explicit(a, x)) <= 1e-15)
        z = M.SparseMatrix.from_triplets(2, 2, [(0, 0, 1.0)])
        with pytest.raises(Exception):
            o.loss_explicit(z, [0.0, 1.0])


def test_spmv_bitwise_port_vs_ref(port, ref):
    a = M.random_sparse(port, 40, 0.2, 11)
    x = port.random_unit_vectors(5, 40)[0]
    assert np.array_equal(port.matvec(a, x), ref.matvec(a, x))
    assert np.array_equal(port.transpose_matvec(a, x), ref.transpose_matvec(a, x))


def test_column_and_row_norms_port_vs_ref(port, ref):
    # column_norms (sparse.hpp:244-268) and row two_norms (row_scale factors)
    mats = [M.random_sparse(port, 50, 0.2, 3), M.row_scaled(M.laplacian2d(12), port, 4),
            M.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 0.0)])]
    n, rp, ci, va = ref.generate_illconditioned(60, 11)
    mats.append(M.SparseMatrix(n, n, rp, ci, va))
    for a in mats:
        assert np.array_equal(port.column_norms(a), ref.column_norms(a))
        assert np.array_equal(port.row_norms(a), ref.row_norms(a))
    a = M.SparseMatrix.from_triplets(2, 2, [(0, 0, 2.0), (1, 1, 3.0)])  # test_sparse.cpp:102-106
    assert list(port.column_norms(a)) == [2.0, 3.0]


@pytest.mark.parametrize("seed", [1, 7])
def test_projected_adam_bitwise_port_vs_ref(port, ref, seed):
    a = M.row_scaled(M.laplacian2d(12), port, seed)
    c = M.cfg(alpha=1e-2, max_iter=600, patience=600, seed=seed)
    e1 = port.projected_adam_explicit(a, c, trace=True)
    e2 = ref.projected_adam_explicit(a, c, trace=True)
    assert e1.value == e2.value and e1.iterations == e2.iterations
    assert e1.converged == e2.converged
    assert np.array_equal(e1.witness, e2.witness)
    assert np.array_equal(e1.trace, e2.trace, equal_nan=True)


def test_estimate_norm_and_cond2_bitwise(port, ref):
    a = M.random_sparse(port, 25, 0.25, 17)
    c = M.cfg(seed=7)
    assert port.estimate_norm_explicit(a, c, 3).value == ref.estimate_norm_explicit(a, c, 3).value
    k1, k2 = port.cond2(a, c), ref.cond2(a, c)
    assert k1["kappa"] == k2["kappa"]
    assert k1["inverse_norm"].iterations == k2["inverse_norm"].iterations


def test_lu_bitwise_port_vs_ref(port, ref):
    a = M.random_sparse(port, 30, 0.3, 5)
    f1, f2 = port.lu_factorize(a, 1e-14), ref.lu_factorize(a, 1e-14)
    e1, e2 = f1.export(), f2.export()
    for k in ("l", "u"):
        for p, q in zip(e1[k], e2[k]):
            assert np.array_equal(p, q)
    assert np.array_equal(e1["row_perm"], e2["row_perm"])
    b = port.random_unit_vectors(2, 30)[0]
    assert np.array_equal(port.lu_solve(f1, b), ref.lu_solve(f2, b))
    assert np.array_equal(port.lu_transpose_solve(f1, b), ref.lu_transpose_solve(f2, b))


def test_lu_singular_cases(oracles):
    # test_condest.cpp:303-326
    dup = M.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (0, 1, 2.0), (1, 0, 1.0), (1, 1, 2.0),
                                              (2, 2, 5.0)])
    empty_col = M.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 0, 1.0)])
    for o in oracles:
        with pytest.raises(Exception) as e:
            o.lu_factorize(dup, 1e-14)
        assert e.value.code == 5
        with pytest.raises(Exception) as e:
            o.lu_factorize(empty_col, 1e-14)
        assert e.value.code == 4
        r = o.cond2(dup, M.cfg())
        assert math.isinf(r["kappa"]) and r["operator_norm"].value > 0


def test_known_norms(oracles):
    # test_condest.cpp:140-160
    for o in oracles:
        e = o.projected_adam_explicit(M.SparseMatrix.identity(10), M.cfg())
        assert abs(e.value - 1.0) <= 1e-12 and e.converged and e.iterations < 2000
        e = o.projected_adam_explicit(M.diag_matrix([3.0, 1.0, 1e-3]), M.cfg())
        assert e.converged and e.value == pytest.approx(3.0, rel=1e-9)
        f = o.lu_factorize(M.diag_matrix([3.0, 1.0, 1e-3]))
        e = o.projected_adam_inverse(f, M.cfg())
        assert e.converged and e.value == pytest.approx(1e3, rel=1e-9)
        z = o.projected_adam_explicit(M.SparseMatrix.from_triplets(4, 4, []), M.cfg())
        assert z.value == 0.0 and not z.converged


def test_singularity_bound_frozen_values(oracles):
    # test_error_bounds.cpp:102-111, acceptance.cpp:192-204
    refs = [(1.0, 2.2204460492503136e-16), (1e6, 2.220446049496832e-10),
            (1e10, 2.2204485144433790e-06), (1e12, 2.2206925956553440e-04)]
    for o in oracles:
        for k, v in refs:
            assert abs(o.singularity_bound(k) - v) / v <= 1e-12
        assert o.singularity_bound(2.0 ** 52) == 2.0
        assert math.isinf(o.singularity_bound(2.0 ** 53))


def test_bounds_endpoints(oracles):
    # test_error_bounds.cpp:44-97
    for o in oracles:
        assert o.loose_bounds(0.0, 2.0, 1e9) == (0.0, 0.0)
        assert o.loose_bounds(0.5, 2.0, 1.0) == (0.25, 0.25)
        assert o.loose_bounds(0.1, 1.0, math.inf) == (0.0, math.inf)
        lo, hi = o.tight_bounds(0.7, 3.0, 2.0, 1.0)
        assert lo == hi and lo == pytest.approx(0.7 / 6.0, rel=1e-15)
        assert o.propagate_bound(0.5) == 1.0 and math.isinf(o.propagate_bound(1.0))
        for args, code in [((0.1, 0.0, 2.0), 6), ((0.1, 1.0, 0.5), 2), ((-0.1, 1.0, 2.0), 2)]:
            with pytest.raises(Exception) as e:
                o.loose_bounds(*args)
            assert e.value.code == code


def test_verify_solution_port_vs_ref(port, ref):
    a = M.random_sparse(port, 20, 0.3, 3)
    x = port.uniform_in(70, 20, -1.0, 1.0)
    b = port.matvec(a, x)
    xh = x + 1e-6 * port.random_unit_vectors(4, 20)[0]
    r1 = port.verify_solution(a, xh, b)
    r2 = ref.verify_solution(a, xh, b)
    assert r1 == r2
    r1 = port.verify_solution(a, xh, b, kappa=50.0, a_norm=3.0)
    r2 = ref.verify_solution(a, xh, b, kappa=50.0, a_norm=3.0)
    assert r1 == r2


@pytest.mark.parametrize("kind,grid,param", [(1, 16, 0), (2, 8, 0), (3, 6, 0), (5, 3000, 256)])
def test_reference_arm_generator_matches_product(kind, grid, param):
    # bench.py's reference arm builds its workload with oracle/_build/libcondkit_gen.so (a g++
    # build of the product's host generator) so that it never loads libcondkit_b200.so; the
    # two builds must emit the same operator bit for bit.
    import pyoracle
    from paper_2409_11515_b200 import configs
    a = pyoracle.generate(kind, grid, 7, param)
    b = configs.generate(kind, grid, 7, param)
    assert a.nrows == b.nrows
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))


def test_optimised_reference_builds_agree(ref):
    # The -O3 builds bench.py times compute the same bits as the
    # -O2 build the golden fixtures come from.
    import pyoracle
    a = M.row_scaled(M.laplacian2d(12), ref, 3)
    cfg = M.cfg(seed=5, max_iter=60, patience=60, alpha=1e-2)
    base = ref.projected_adam_explicit(a, cfg, trace=True)
    flags = pyoracle._cpu_flags()
    for which in ("ref_v3", "ref_native"):
        if not pyoracle.available(which) or (which == "ref_native" and
                                             pyoracle.best_reference() != "ref_native"):
            continue
        if which == "ref_v3" and not {"avx2", "fma", "bmi2"} <= flags:
            continue
        e = pyoracle.Oracle(which).projected_adam_explicit(a, cfg, trace=True)
        assert e.value == base.value and e.iterations == base.iterations
        assert np.array_equal(e.witness, base.witness)
        assert np.array_equal(e.trace, base.trace)
