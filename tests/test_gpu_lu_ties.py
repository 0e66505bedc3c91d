"""lu_factorize on the device vs the oracle where the pivot rule's details
matter: magnitude ties (broken by the reference's touched order, lu.hpp:88-124),
structural vs numerical singularity (lu.hpp:126-129), explicit zeros, and bands
too wide for the panel multipliers to sit in shared memory (any pattern up to
the solve window). Factors are compared in the reference's LUFactors shape
(L/U CSR, row_perm, pivot_min), bit for bit."""
import numpy as np
import pytest

import paper_2409_11515_b200 as ck
from test_gpu_inverse import assert_same_factors

pytestmark = pytest.mark.gpu


def csr(n, entries):
    """CSR from (row, col, value) keeping explicit zeros (SparseMatrix stores them)."""
    entries = sorted(entries)
    rp = np.zeros(n + 1, np.int64)
    for r, _, _ in entries:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    ci = np.array([c for _, c, _ in entries], np.int32)
    va = np.array([v for _, _, v in entries], np.float64)
    return ck.SparseMatrix(n, n, rp, ci, va)


def factor_both(port, a, tol=1e-12):
    """(device factors or exception, oracle factors or exception)."""
    try:
        rf = port.lu_factorize(a, tol)
        rerr = None
    except Exception as e:  # noqa: BLE001
        rf, rerr = None, e
    try:
        f = ck.lu_factorize(a, tol)
        err = None
    except (ck.StructurallySingular, ck.NumericallySingular) as e:
        f, err = None, e
    return f, err, rf, rerr


def check_same(port, a, tol=1e-12):
    f, err, rf, rerr = factor_both(port, a, tol)
    if rerr is not None:
        # oracle status 4 = StructurallySingular, 5 = NumericallySingular (lu.hpp:24-40)
        assert err is not None, f"oracle raised {rerr}, device factored"
        want = ck.StructurallySingular if rerr.code == 4 else ck.NumericallySingular
        assert isinstance(err, want), (err, rerr)
        assert err.column == rerr.column
        return "singular"
    assert err is None, f"device raised {err}, oracle factored"
    assert_same_factors(f, rf, a)
    return "ok"


def test_tie_goes_to_first_touched_row(port):
    # column 0 = rows 0, 1, 3 (1, 1, 4) pivots on row 3; column 1 then has
    # original row 0 (2 - 0.25 * 4 = 1) and fill row 1 (0 - 0.25 * 4 = -1): equal
    # magnitudes, and the reference takes the original entry (row 0) -- not the
    # lowest band position (row 1).
    a = csr(4, [(0, 0, 1.0), (0, 1, 2.0), (0, 2, 1.0),
                (1, 0, 1.0), (1, 2, 3.0), (1, 3, 1.0),
                (2, 2, 1.0), (2, 3, 2.0),
                (3, 0, 4.0), (3, 1, 4.0), (3, 3, 1.0)])
    assert check_same(port, a) == "ok"
    assert int(ck.lu_factorize(a).row_perm[1]) == 0


@pytest.mark.parametrize("n,density,seed", [(6, 0.5, 1), (12, 0.3, 2), (30, 0.15, 3),
                                            (64, 0.08, 4), (100, 0.05, 5), (150, 0.04, 6),
                                            (200, 0.02, 7)])
def test_integer_matrices_bitwise(port, n, density, seed):
    # entries in {-2, -1, 1, 2}: pivot ties on almost every column, fill-vs-original and
    # fill-vs-fill orders both exercised; several draws per shape
    rng = np.random.default_rng(seed)
    outcomes = []
    for _ in range(6):
        ent = {}
        for i in range(n):
            ent[(i, int(rng.integers(n)))] = float(rng.choice([-2, -1, 1, 2]))
            for j in np.nonzero(rng.random(n) < density)[0]:
                ent[(i, int(j))] = float(rng.choice([-2, -1, 1, 2]))
        a = csr(n, [(r, c, v) for (r, c), v in ent.items()])
        outcomes.append(check_same(port, a))
    assert "ok" in outcomes


def test_structural_vs_numerical_singularity(port):
    # column 1's only touched row (row 0) is pivoted in column 0, and column 0's
    # multipliers reach no other row: structural (lu.hpp:126)
    a = csr(3, [(0, 0, 2.0), (0, 1, 1.0), (1, 2, 1.0), (2, 2, 1.0)])
    f, err, rf, rerr = factor_both(port, a)
    assert isinstance(err, ck.StructurallySingular) and rerr.code == 4
    assert err.column == 1
    # the same with an explicit zero in an unpivoted row: a candidate of magnitude 0,
    # numerically singular (lu.hpp:127)
    b = csr(3, [(0, 0, 2.0), (0, 1, 1.0), (1, 2, 1.0), (2, 1, 0.0), (2, 2, 1.0)])
    f, err, rf, rerr = factor_both(port, b)
    assert isinstance(err, ck.NumericallySingular) and rerr.code == 5
    assert err.column == 1
    # an empty column
    c = csr(3, [(0, 0, 1.0), (1, 0, 1.0), (2, 2, 1.0), (1, 2, 3.0)])
    assert check_same(port, c) == "singular"
    # fill reaching an otherwise empty position keeps a column factorable
    d = csr(3, [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 1.0), (2, 2, 1.0), (1, 2, 1.0)])
    assert check_same(port, d) == "ok"


def test_cond2_maps_both_singularities_to_infinity():
    a = csr(3, [(0, 0, 2.0), (0, 1, 1.0), (1, 2, 1.0), (2, 2, 1.0)])
    r = ck.cond2(a, ck.AdamConfig(max_iter=50, patience=50), 1)
    assert r.kappa == float("inf") and r.inverse_norm.value == float("inf")


def test_full_width_band_factors_and_cond2(port):
    # a random sparse n = 2000 matrix whose pattern spans the whole matrix
    # (kl, ku ~ n): the panel multipliers no longer fit shared memory and are read from
    # the band; factors and cond2 against the oracle (lu.hpp:55-177, condest.hpp:341-365)
    n = 2000
    rng = np.random.default_rng(11)
    ent = {(i, i): float(rng.uniform(0.5, 1.5)) for i in range(n)}
    for i in range(n):
        for j in rng.integers(0, n, 5):
            ent[(i, int(j))] = float(rng.uniform(-1.0, 1.0))
    ent[(n - 1, 0)] = 0.5
    ent[(0, n - 1)] = -0.5
    a = csr(n, [(r, c, v) for (r, c), v in ent.items()])
    f = ck.lu_factorize(a, 1e-14)
    assert f.kl == n - 1 and f.ku == n - 1
    rf = port.lu_factorize(a, 1e-14)
    assert_same_factors(f, rf)
    cfg = ck.AdamConfig(alpha=1e-2, max_iter=200, patience=200, seed=3)
    r = ck.cond2(a, cfg, 1, 1e-14)
    g = port.cond2(a, cfg, 1, 1e-14)
    assert r.kappa == pytest.approx(g["kappa"], rel=1e-3)
    assert r.inverse_norm.value == pytest.approx(g["inverse_norm"].value, rel=1e-9)
    assert r.operator_norm.value == pytest.approx(g["operator_norm"].value, rel=1e-12)


def test_band_limit_reported_before_allocation():
    # kl + ku beyond the solve window: a clear UNSUPPORTED status, nothing allocated
    n = 20000
    a = csr(n, [(i, i, 1.0) for i in range(n)] + [(n - 1, 0, 1.0), (0, n - 1, 1.0)])
    with pytest.raises(ck.CondkitError, match="band too wide"):
        ck.lu_factorize(a)


def test_batched_factorisation_matches_single(port):
    # ck_lu_factorize_batch with members of different band widths (each member's key
    # window is its own): factors identical to separate factorisations and the oracle
    from paper_2409_11515_b200 import batch, configs
    rng = np.random.default_rng(21)
    mem = [configs.ensemble_member(0, 1, n=1000, bw=64), configs.ensemble_member(1, 1, n=513, bw=40),
           configs.ensemble_member(2, 1, n=700, bw=200)]
    for n in (40, 90):
        ent = {(i, int(rng.integers(n))): float(rng.choice([-2, -1, 1, 2])) for i in range(n)}
        for i in range(n):
            ent[(i, i)] = float(rng.choice([-2, -1, 1, 2]))
            for j in np.nonzero(rng.random(n) < 0.08)[0]:
                ent[(i, int(j))] = float(rng.choice([-2, -1, 1, 2]))
        mem.append(csr(n, [(r, c, v) for (r, c), v in ent.items()]))
    facs = batch.lu_factorize_many(mem, 1e-14)
    for m, f in zip(mem, facs):
        try:
            rf = port.lu_factorize(m, 1e-14)
        except Exception:  # noqa: BLE001
            assert isinstance(f, (ck.StructurallySingular, ck.NumericallySingular))
            continue
        assert_same_factors(f, rf)
        assert_same_factors(ck.lu_factorize(m, 1e-14), rf)
