"""Row-block partition on the device: every rank's sessions in
one process on one GPU (lockstep, device copies for the collectives) and the
NCCL backend at world size 1, against the single-device loop and the oracle.
The sparse products are bit-identical; the reductions merge per-rank partials
in rank order, so results agree to rounding, not bitwise."""
import numpy as np
import pytest

import matrices as M
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs, dist

pytestmark = pytest.mark.gpu


def _mats(port):
    return {"laplacian": M.row_scaled(M.laplacian2d(48), port, 1),
            "random": M.random_sparse(port, 700, 0.01, 5),
            "banded": configs.ensemble_member(0, 1, n=4000, bw=120),
            "hm": configs.generate(3, 12)}


@pytest.mark.parametrize("kind", ["laplacian", "random", "banded", "hm"])
@pytest.mark.parametrize("P", [1, 2, 3])
def test_partition_matches_single_device(port, kind, P):
    a = _mats(port)[kind]
    cfg = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=3)
    got = dist.projected_adam_partitioned(a, P, cfg, seeds=[3, 4])
    for e, sd in zip(got, [3, 4]):
        c = M.cfg(alpha=1e-2, max_iter=300, patience=300, seed=sd)
        one = ck.projected_adam(ck.ExplicitOracle(a), c)
        o = port.projected_adam_explicit(a, c)
        assert e.iterations == one.iterations == o.iterations
        assert e.value == pytest.approx(one.value, rel=1e-10)
        assert e.value == pytest.approx(o.value, rel=1e-9)
        assert np.linalg.norm(port.matvec(a, e.witness)) == pytest.approx(e.value, rel=1e-12)
        assert abs(np.linalg.norm(e.witness) - 1.0) < 1e-12


def test_partition_default_patience_and_restarts(port):
    # early stopping and degenerate restarts decided identically on every rank
    a = M.random_sparse(port, 500, 0.01, 9)
    cfg = M.cfg(seed=2)
    got = dist.projected_adam_partitioned(a, 3, cfg)[0]
    o = port.projected_adam_explicit(a, cfg)
    assert got.iterations == o.iterations and got.converged == o.converged
    assert got.value == pytest.approx(o.value, rel=1e-9)


def test_partition_timing_and_lists(port):
    a = configs.generate(3, 16)
    parts = dist.build_partition(a, 4)
    for p in parts:  # halo lists pair up
        for q in parts:
            if p.rank == q.rank:
                continue
            ns = p.lists["xs_off"][q.rank + 1] - p.lists["xs_off"][q.rank]
            nr = q.lists["xr_off"][p.rank + 1] - q.lists["xr_off"][p.rank]
            assert ns == nr
    s = dist.PartitionedSession(parts, M.cfg(alpha=1e-2, max_iter=10**6, patience=10**6), [1])
    s.run(3)
    assert s.time(5) > 0.0


def test_nccl_backend_single_rank(port):
    a = configs.generate(3, 12)
    parts = dist.build_partition(a, 1)
    cfg = M.cfg(alpha=1e-2, max_iter=200, patience=200, seed=5)
    s = dist.PartitionedSession(parts, cfg, [5], nranks=1, nccl_id=dist.nccl_unique_id())
    assert s.run()
    e = s.result(0, 0)
    one = ck.projected_adam(ck.ExplicitOracle(a), cfg)
    assert e.iterations == one.iterations
    assert e.value == pytest.approx(one.value, rel=1e-12)
    assert s.time(3) > 0.0


@pytest.mark.parametrize("kind", ["hm", "banded"])
def test_partition_eight_ranks(port, kind):
    """BASELINE's 8-rank row-block partition, all ranks in one process: one exchange
    (partials + halo) per half step framed by the fused pack / combine kernels."""
    a = {"hm": lambda: configs.generate(3, 24), "banded": lambda: configs.ensemble_member(2, 1, n=6000, bw=100)}[kind]()
    cfg = M.cfg(alpha=1e-2, max_iter=200, patience=200, seed=7)
    got = dist.projected_adam_partitioned(a, 8, cfg, seeds=[7, 8])
    for e, sd in zip(got, [7, 8]):
        c = M.cfg(alpha=1e-2, max_iter=200, patience=200, seed=sd)
        one = ck.projected_adam(ck.ExplicitOracle(a), c)
        assert e.iterations == one.iterations
        assert e.value == pytest.approx(one.value, rel=1e-10)
        assert np.linalg.norm(port.matvec(a, e.witness)) == pytest.approx(e.value, rel=1e-12)
