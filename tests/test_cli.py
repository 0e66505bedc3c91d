"""tools/condkit_b200_cli: the reference CLI's cond / norm / verify
(condkit_cli.cpp:141-326) on the device, and `convert` to binary CSR.
Matrix Market parsing is pinned to the reference's own reader; the
estimator outputs to the oracle with the CLI's defaults (alpha 0.05,
patience 100, restarts 3)."""
import os
import subprocess

import numpy as np
import pytest

import matrices as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "condkit_b200_cli")

MM_CASES = {
    "coord_general_dups": "%%MatrixMarket matrix coordinate real general\n% c\n\n3 4 6\n1 1 2.5\n2 3 -1e-3\n"
                          "1 1 0.5\n3 4 7\n2 1 +4\n3 2 -0.125\n",
    "coord_symmetric_int": "%%MatrixMarket matrix coordinate integer symmetric\n4 4 5\n1 1 4\n2 1 -1\n"
                           "3 3 5\n4 2 2\n4 4 9\n",
    "array_general": "%%MatrixMarket matrix array real general\n2 3\n1\n0\n0.5\n2\n0\n-3\n",
    "array_symmetric": "%%MatrixMarket matrix array real symmetric\n3 3\n4\n-1\n0\n5\n2\n6\n",
}


def _run(*args, check=True):
    p = subprocess.run([CLI, *args], capture_output=True, text=True)
    if check and p.returncode not in (0, 3, 4):
        raise AssertionError(p.stderr)
    return p


def _kv(out: str) -> dict:
    d = {}
    for line in out.splitlines():
        if line.startswith("#") or " = " not in line:
            continue
        k, v = line.split(" = ", 1)
        d[k] = v
    return d


def _read_csrb(path):
    with open(path, "rb") as f:
        assert f.read(8) == b"CKCSR001"
        nr, nc, nnz = np.frombuffer(f.read(24), np.int64)
        rp = np.frombuffer(f.read(8 * (nr + 1)), np.int64)
        ci = np.frombuffer(f.read(4 * nnz), np.int32)
        va = np.frombuffer(f.read(8 * nnz), np.float64)
    return int(nr), int(nc), rp, ci, va


def _write_mm(path, a):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{a.nrows} {a.ncols} {a.nnz}\n")
        rp, ci, va = a.row_offsets, a.col_indices, a.values
        for i in range(a.nrows):
            for k in range(rp[i], rp[i + 1]):
                f.write(f"{i + 1} {ci[k] + 1} {float(va[k])!r}\n")


@pytest.mark.parametrize("case", sorted(MM_CASES))
def test_convert_matches_reference_reader(tmp_path, ref, case):
    src = tmp_path / "a.mtx"
    src.write_text(MM_CASES[case])
    out = tmp_path / "a.csrb"
    p = _run("convert", "--matrix", str(src), "--out", str(out))
    assert p.returncode == 0
    got = _read_csrb(out)
    want = ref.read_matrix_market(str(src))
    assert got[0] == want[0] and got[1] == want[1]
    for g, w in zip(got[2:], want[2:]):
        assert np.array_equal(g, w)


def test_parse_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 2.0\n")
    p = _run("convert", "--matrix", str(bad), "--out", str(tmp_path / "x.csrb"), check=False)
    assert p.returncode == 2 and "parse error" in p.stderr
    p = _run("frobnicate", check=False)
    assert p.returncode == 2


@pytest.mark.gpu
def test_cond_norm_verify_vs_oracle(tmp_path, port):
    a = M.random_sparse(port, 60, 0.15, 8)
    mtx = tmp_path / "a.mtx"
    _write_mm(mtx, a)
    csrb = tmp_path / "a.csrb"
    _run("convert", "--matrix", str(mtx), "--out", str(csrb))
    cfg = M.cfg(alpha=0.05, max_iter=2000, patience=100, rel_tol=1e-12, seed=1)
    o = port.cond2(a, cfg, restarts=3)
    for src in (mtx, csrb):
        p = _run("cond", "--matrix", str(src))
        d = _kv(p.stdout)
        assert p.returncode == (3 if o["kappa"] >= 2.0 ** 53 else 0)
        assert float(d["kappa2"]) == pytest.approx(o["kappa"], rel=1e-9)
        assert float(d["operator_norm_recomputed"]) == pytest.approx(float(d["operator_norm"]), rel=1e-12)
        assert float(d["inverse_norm_recomputed"]) == pytest.approx(float(d["inverse_norm"]), rel=1e-12)
        assert int(d["n"]) == 60 and int(d["nnz"]) == a.nnz
    p = _run("norm", "--matrix", str(csrb), "--restarts", "2", "--seed", "7")
    d = _kv(p.stdout)
    on = port.estimate_norm_explicit(a, M.cfg(alpha=0.05, max_iter=2000, patience=100, seed=7), 2)
    assert float(d["operator_norm"]) == pytest.approx(on.value, rel=1e-9)
    assert int(d["iterations"]) == on.iterations
    # verify: b = A x*, xhat = x* + small perturbation
    x = port.uniform_in(70, 60, -1.0, 1.0)
    b = port.matvec(a, x)
    xh = x + 1e-9 * port.random_unit_vectors(4, 60)[0]
    for name, v in (("b.txt", b), ("x.txt", xh)):
        (tmp_path / name).write_text("# vec\n" + "\n".join(repr(float(t)) for t in v) + "\n")
    p = _run("verify", "--matrix", str(mtx), "--rhs", str(tmp_path / "b.txt"), "--solution",
             str(tmp_path / "x.txt"), "--threshold", "1e-3")
    d = _kv(p.stdout)
    ro = port.verify_solution(a, xh, b, threshold=1e-3,
                              adam=M.cfg(alpha=0.05, max_iter=2000, patience=100, seed=1))
    assert d["verdict"] == ["accepted", "rejected", "numerically_singular"][ro["verdict"]]
    assert float(d["residual_norm"]) == pytest.approx(ro["residual_norm"], rel=1e-13)
    assert float(d["tight_upper"]) == pytest.approx(ro["tight_upper"], rel=1e-9)
    assert p.returncode == {"accepted": 0, "numerically_singular": 3, "rejected": 4}[d["verdict"]]


@pytest.mark.gpu
def test_cond_column_scaling_drops_kappa(tmp_path, ref):
    n, rp, ci, va = ref.generate_illconditioned(300, 2)
    a = M.SparseMatrix(n, n, rp, ci, va)
    mtx = tmp_path / "a.mtx"
    _write_mm(mtx, a)
    k0 = float(_kv(_run("cond", "--matrix", str(mtx)).stdout)["kappa2"])
    k1 = float(_kv(_run("cond", "--matrix", str(mtx), "--scale", "column").stdout)["kappa2"])
    assert k0 / k1 >= 1e10


def test_csrb_python_roundtrip(tmp_path, port):
    from paper_2409_11515_b200 import csrb
    a = M.random_sparse(port, 90, 0.1, 4)
    p = tmp_path / "a.csrb"
    csrb.write_csrb(a, str(p))
    b = csrb.read_csrb(str(p))
    assert np.array_equal(b.row_offsets, a.row_offsets) and np.array_equal(b.values, a.values)
    mtx = tmp_path / "a.mtx"
    _write_mm(mtx, a)
    out = tmp_path / "b.csrb"
    _run("convert", "--matrix", str(mtx), "--out", str(out))
    c = csrb.read_csrb(str(out))
    assert np.array_equal(c.col_indices, a.col_indices) and np.array_equal(c.values, a.values)
