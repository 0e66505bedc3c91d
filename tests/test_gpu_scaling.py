"""Column / row scaling on the device (sparse.hpp:244-313) vs the reference,
and acceptance criterion 5 (acceptance.cpp:209-230): column scaling drops the
generator's kappa by >= 1e10."""
import numpy as np
import pytest

import matrices as M
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs

pytestmark = pytest.mark.gpu


def _mats(port, ref):
    n, rp, ci, va = ref.generate_illconditioned(200, 11)
    return {"random": M.random_sparse(port, 80, 0.1, 3),
            "rowscaled": M.row_scaled(M.laplacian2d(20), port, 2),
            "c5member": configs.ensemble_member(2, 1, n=3000, bw=100),
            "twoplateau": ck.SparseMatrix(n, n, rp, ci, va),
            "rect": ck.SparseMatrix.from_triplets(3, 5, [(0, 4, 2.0), (1, 0, -1.0), (2, 2, 7.0),
                                                         (0, 0, 1e-300), (2, 4, 3.0)])}


@pytest.mark.parametrize("kind", ["random", "rowscaled", "c5member", "twoplateau", "rect"])
def test_norms_bitwise(port, ref, kind):
    a = _mats(port, ref)[kind]
    assert np.array_equal(ck.column_norms(a), ref.column_norms(a))
    assert np.array_equal(ck.row_norms(a), ref.row_norms(a))


def test_known_answers_and_zero_column():
    # test_sparse.cpp:102-126
    a = ck.SparseMatrix.from_triplets(2, 2, [(0, 0, 2.0), (1, 1, 3.0)])
    assert list(ck.column_norms(a)) == [2.0, 3.0]
    s, d = ck.column_scale(a)
    assert s.coeff(0, 0) == 1.0 and s.coeff(1, 1) == 1.0 and d[0] == 2.0 and d[1] == 3.0
    z = ck.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 0.0)])
    with pytest.raises(ck.ZeroColumn) as e:
        ck.column_scale(z)
    assert e.value.column == 2
    with pytest.raises(ck.ZeroRow) as e:
        ck.row_scale(z, np.ones(3))
    assert e.value.row == 2


def test_column_scale_values_and_unit_norms(port, ref):
    mats = _mats(port, ref)
    with pytest.raises(ck.ZeroColumn) as e:  # columns 1 and 3 are empty
        ck.column_scale(mats.pop("rect"))
    assert e.value.column == 1
    for a in mats.values():
        s, d = ck.column_scale(a)
        want = a.values / ref.column_norms(a)[a.col_indices]  # vals[k] /= norms[cols[k]]
        assert np.array_equal(s.values, want)
        assert np.array_equal(s.row_offsets, a.row_offsets)
        for v in ck.column_norms(s):
            assert abs(v - 1.0) <= 1e-14


def test_row_scale_and_unscale(port, ref):
    a = _mats(port, ref)["random"]
    b = port.uniform_in(3, a.nrows, -1.0, 1.0)
    s, bs = ck.row_scale(a, b)
    rn = ref.row_norms(a)
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_offsets))
    assert np.array_equal(s.values, a.values / rn[rows])
    assert np.array_equal(bs, b / rn)
    # test_sparse.cpp:128-145: the column-scaled system recovers the solution
    a = M.random_sparse(port, 20, 0.3, 21)
    xt = port.random_unit_vectors(5, 20)[0]
    bb = port.matvec(a, xt)
    sa, d = ck.column_scale(a)
    y = np.linalg.solve(sa.to_dense(), bb)
    x = ck.unscale_solution(y, d)
    assert np.array_equal(x, y / d.factors)
    assert np.allclose(x, np.linalg.solve(a.to_dense(), bb), atol=1e-10)


def test_criterion5_column_scaling_drops_kappa(port, ref):
    # acceptance.cpp:219-229 at n = 500, seed 2 (the reference's own recipe)
    n, rp, ci, va = ref.generate_illconditioned(500, 2)
    a = ck.SparseMatrix(n, n, rp, ci, va)
    before = ck.cond2(a).kappa
    s, _ = ck.column_scale(a)
    after = ck.cond2(s).kappa
    assert np.isfinite(before) and before / after >= 1e10
    o = port.cond2(s, M.cfg())
    assert after == pytest.approx(o["kappa"], rel=1e-3)
