"""SpMV parity through the C-ABI against the oracle (bit-exact: the device sums
each row in stored order with unfused multiply/add, exactly matvec /
transpose_matvec, sparse.hpp:212-242)."""
import numpy as np
import pytest

import matrices as M
import paper_2409_11515_b200 as ck

pytestmark = pytest.mark.gpu


def _cases(port):
    yield "random20", M.random_sparse(port, 20, 0.3, 11)
    yield "random100", M.random_sparse(port, 100, 0.1, 12)
    yield "laplacian_rowscaled", M.row_scaled(M.laplacian2d(33), port, 1)
    yield "identity", ck.SparseMatrix.identity(7)
    rng = np.random.default_rng(5)
    # ragged rows incl. empty rows and one long row, rectangular
    r, c = [], []
    for i in range(700):
        k = 0 if i % 17 == 0 else (300 if i == 5 else rng.integers(1, 12))
        cols = np.sort(rng.choice(1000, size=k, replace=False))
        r += [i] * k
        c += list(cols)
    yield "ragged_rect", ck.SparseMatrix.from_coo(700, 1000, r, c, rng.standard_normal(len(r)))
    yield "empty", ck.SparseMatrix.from_triplets(5, 3, [])


def test_matvec_bitwise(port):
    for name, a in _cases(port):
        x = port.random_unit_vectors(3, a.ncols)[0] if a.ncols else np.zeros(0)
        y = ck.matvec(a, x)
        assert np.array_equal(y, port.matvec(a, x)), name
        u = port.random_unit_vectors(4, a.nrows)[0] if a.nrows else np.zeros(0)
        z = ck.transpose_matvec(a, u)
        assert np.array_equal(z, port.transpose_matvec(a, u)), name


def test_matvec_matches_dense_and_adjoint(port):
    # test_sparse.cpp:57-84
    for seed in (11, 12, 13):
        a = M.random_sparse(port, 20, 0.3, seed)
        d = a.to_dense()
        x = port.random_unit_vectors(seed + 100, 20)[0]
        assert np.allclose(ck.matvec(a, x), d @ x, atol=1e-13, rtol=0)
        assert np.allclose(ck.transpose_matvec(a, x), d.T @ x, atol=1e-13, rtol=0)
    a = M.random_sparse(port, 20, 0.25, 7)
    xs = port.random_unit_vectors(99, 20, 20)
    for k in range(10):
        x, y = xs[2 * k], xs[2 * k + 1]
        assert abs(y @ ck.matvec(a, x) - x @ ck.transpose_matvec(a, y)) <= 1e-13


def test_basis_vectors_reproduce_columns(port):
    # test_sparse.cpp:86-94
    a = M.random_sparse(port, 10, 0.4, 3)
    for j in range(10):
        e = np.zeros(10)
        e[j] = 1.0
        col = ck.matvec(a, e)
        for i in range(10):
            assert col[i] == a.coeff(i, j)


def test_dimension_mismatch():
    a = ck.SparseMatrix.identity(3)
    with pytest.raises(ck.DimensionMismatch):
        ck.matvec(a, [1.0, 2.0])
    with pytest.raises(ck.DimensionMismatch):
        ck.transpose_matvec(a, [1.0, 2.0])


def test_device_validation_rejects_bad_csr():
    # bypass host validation: the device check must still catch it
    bad = ck.SparseMatrix(2, 2, [0, 2, 3], [1, 0, 1], [1.0, 2.0, 3.0], validate=False)
    with pytest.raises(ck.DimensionMismatch):
        bad.device()


def test_residual_norms(port):
    a = M.random_sparse(port, 50, 0.2, 9)
    x = port.uniform_in(70, 50, -1.0, 1.0)
    b = port.matvec(a, x) + 1e-3
    rn, xn, bn = a.device().residual_norms(x, b)
    r = port.matvec(a, x) - b
    assert rn == pytest.approx(port.two_norm(r), rel=1e-14)
    assert xn == pytest.approx(port.two_norm(x), rel=1e-15)
    assert bn == pytest.approx(port.two_norm(b), rel=1e-15)


def test_norm_overflow_safety():
    # two_norm overflow safety (test_sparse.cpp:49-54) on the device reduction
    a = ck.SparseMatrix.identity(25)
    x = np.full(25, 1e300)
    rn, xn, bn = a.device().residual_norms(x, np.full(25, 3e300))
    assert xn == pytest.approx(5e300, rel=1e-15)
    assert bn == pytest.approx(15e300, rel=1e-15)
    assert rn == pytest.approx(10e300, rel=1e-15)


def _wide_span_matrix():
    # one entry per row at column 2200 i: a 32-row slice of A spans 68200 > 65535
    # columns (wide int32 format), while every slice of A^T stays narrow.
    n_r, n_c = 1000, 2200 * 999 + 1
    rows = np.arange(n_r)
    vals = np.random.default_rng(3).standard_normal(n_r)
    return ck.SparseMatrix.from_coo(n_r, n_c, rows, 2200 * rows, vals)


def test_column_formats_and_bitwise(port, monkeypatch):
    """The narrow (uint16 offset) and wide (int32) column formats give identical
    bits; a slice spanning >= 65536 columns falls back to wide per operator."""
    a = M.row_scaled(M.laplacian2d(40), port, 2)
    x = port.random_unit_vectors(8, a.ncols)[0]
    want_y, want_z = port.matvec(a, x), port.transpose_matvec(a, x)
    assert a.device().info()["col_format"] & 3 == 3
    assert np.array_equal(ck.matvec(a, x), want_y)
    assert np.array_equal(ck.transpose_matvec(a, x), want_z)
    monkeypatch.setenv("CK_SELL_WIDE", "1")
    w = ck.SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, a.values)
    assert w.device().info()["col_format"] == 0
    assert np.array_equal(ck.matvec(w, x), want_y)
    assert np.array_equal(ck.transpose_matvec(w, x), want_z)
    monkeypatch.delenv("CK_SELL_WIDE")
    m = _wide_span_matrix()
    assert m.device().info()["col_format"] & 3 == 2  # A wide, A^T narrow
    xm = port.random_unit_vectors(9, m.ncols)[0]
    um = port.random_unit_vectors(10, m.nrows)[0]
    assert np.array_equal(ck.matvec(m, xm), port.matvec(m, xm))
    assert np.array_equal(ck.transpose_matvec(m, um), port.transpose_matvec(m, um))


def test_adam_identical_across_column_formats(port, monkeypatch):
    """projected_adam on the narrow and wide layouts: same bits, same iterations."""
    from paper_2409_11515_b200 import configs
    a = configs.generate(configs.LAPLACIAN, 24, 1)
    cfg = configs.baseline_adam(1, max_iter=150)
    e1 = ck.norm2(a, cfg)
    monkeypatch.setenv("CK_SELL_WIDE", "1")
    w = ck.SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, a.values)
    assert w.device().info()["col_format"] == 0
    e2 = ck.norm2(w, cfg)
    assert e1.iterations == e2.iterations
    assert e1.value == e2.value
    assert np.array_equal(e1.witness, e2.witness)


def test_cuda_errors_do_not_linger(port):
    """A CUDA error reported by one call must not resurface in the next (the runtime's
    per-thread last error is cleared), and pinning a pinned range again is benign."""
    import ctypes
    from paper_2409_11515_b200 import _lib
    lib = _lib.load()
    _lib.ensure_device()
    buf = np.arange(1 << 16, dtype=np.float64)
    assert lib.ck_host_register(buf.ctypes.data, buf.nbytes) == 0
    assert lib.ck_host_register(buf.ctypes.data, buf.nbytes) == 0  # already registered
    other = np.zeros(16)
    assert lib.ck_host_unregister(ctypes.c_void_p(other.ctypes.data)) != 0  # never registered: an error...
    a = M.laplacian2d(12)
    x = port.random_unit_vectors(2, a.ncols)[0]
    assert np.array_equal(ck.matvec(a, x), port.matvec(a, x))  # ...that the next call does not see
    assert lib.ck_host_unregister(ctypes.c_void_p(buf.ctypes.data)) == 0


def test_pattern_dictionary_is_invisible(port, monkeypatch):
    """Stencil operators repeat a few slice patterns: their uint16 offsets come from a
    shared table (col_format bits 2 / 3, 8 B per stored entry). Same columns in the same
    order: products and a whole projected_adam run are bit-identical to the per-entry
    offsets (CK_SELL_PATTERN=0); an operator without repeating patterns keeps them."""
    from paper_2409_11515_b200 import configs
    for a in (configs.generate(3, 128), configs.generate(2, 128), configs.generate(configs.LAPLACIAN, 256, 1)):
        x = port.random_unit_vectors(3, a.ncols)[0]
        u = port.random_unit_vectors(4, a.nrows)[0]
        info = a.device().info()
        assert info["col_format"] == 15, info
        y, z = ck.matvec(a, x), ck.transpose_matvec(a, u)
        assert np.array_equal(y, port.matvec(a, x)) and np.array_equal(z, port.transpose_matvec(a, u))
        cfg = configs.baseline_adam(1, max_iter=120)
        e1 = ck.norm2(a, cfg)
        monkeypatch.setenv("CK_SELL_PATTERN", "0")
        b = ck.SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, a.values)
        binfo = b.device().info()
        assert binfo["col_format"] == 3 and binfo["device_bytes"] > info["device_bytes"]
        assert np.array_equal(ck.matvec(b, x), y) and np.array_equal(ck.transpose_matvec(b, u), z)
        e2 = ck.norm2(b, cfg)
        monkeypatch.delenv("CK_SELL_PATTERN")
        assert e1.value == e2.value and e1.iterations == e2.iterations
        assert np.array_equal(e1.witness, e2.witness)
    r = configs.ensemble_member(0, 1, n=20000)  # random in-band columns: no repeating patterns
    assert r.device().info()["col_format"] == 3
