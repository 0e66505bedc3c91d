#!/usr/bin/env python
"""Generates the committed golden fixtures of tests/golden/ by running the
UNMODIFIED reference (oracle/_ref/libcondkit_ref.so, built from
/root/reference/proj/include by oracle/Makefile) on the seeded synthetic
workloads of paper_2409_11515_b200.configs. TEST INFRASTRUCTURE.

    python tests/golden/make_golden.py quick        # minutes
    python tests/golden/make_golden.py c3_sigma_max # ~10 min (2000 reference iterations)
    python tests/golden/make_golden.py c4_sigma_max # ~3 h
    python tests/golden/make_golden.py c2_cond2     # LU at n=196k + 2000 inverse iterations

Each job writes tests/golden/<job>.json. The GPU box never reads
/root/reference; it only reads these files.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402

from paper_2409_11515_b200 import configs  # noqa: E402


def _est(e):
    return {"value": e.value, "iterations": int(e.iterations), "converged": bool(e.converged)}


def _save(name, data):
    data["generated_by"] = "tests/golden/make_golden.py " + name + " (oracle/_ref: the reference)"
    with open(os.path.join(HERE, name + ".json"), "w") as f:
        json.dump(data, f, indent=1)
    print("wrote", name, flush=True)


def spmv_checksums(ref, a, seed=7, samples=257):
    x = ref.random_unit_vectors(seed, a.ncols)[0]
    y = ref.matvec(a, x)
    z = ref.transpose_matvec(a, ref.random_unit_vectors(seed + 1, a.nrows)[0])
    idx_y = np.linspace(0, a.nrows - 1, samples).astype(np.int64)
    idx_z = np.linspace(0, a.ncols - 1, samples).astype(np.int64)
    return {"x_seed": seed, "y_two_norm": ref.two_norm(y), "z_two_norm": ref.two_norm(z),
            "y_idx": idx_y.tolist(), "y_val": [float(v) for v in y[idx_y]],
            "z_idx": idx_z.tolist(), "z_val": [float(v) for v in z[idx_z]]}


def quick(ref):
    out = {}
    cfg = configs.baseline_adam(1)
    # config 1 at full size: single runs, restarts, cond2 (3 restarts each norm)
    a = configs.config(1)
    e = ref.projected_adam_explicit(a, cfg, trace=True)
    out["c1_projected_adam"] = {**_est(e), "first_losses": [float(v) for v in e.trace[:20]]}
    out["c1_estimate_norm3"] = _est(ref.estimate_norm_explicit(a, cfg, 3))
    t0 = time.time()
    c = ref.cond2(a, cfg, 3, 1e-14)
    out["c1_cond2"] = {"kappa": c["kappa"], "operator_norm": _est(c["operator_norm"]),
                       "inverse_norm": _est(c["inverse_norm"]), "seconds": time.time() - t0}
    f = ref.lu_factorize(a, 1e-14)
    out["c1_inv_projected_adam"] = _est(ref.projected_adam_inverse(
        f, configs.baseline_adam(ref.mix_seed(1, 0x1234))))
    # config 2 operator on a 32x32 grid: cond2 and the forward-error bound
    s = configs.generate(configs.STOKES, 32, 1)
    c = ref.cond2(s, cfg, 1, 1e-14)
    out["c2_grid32_cond2_r1"] = {"kappa": c["kappa"], "operator_norm": _est(c["operator_norm"]),
                                 "inverse_norm": _est(c["inverse_norm"])}
    xs = ref.uniform_in(17, s.ncols, -1.0, 1.0)
    b = ref.matvec(s, xs)
    u = ref.random_unit_vectors(19, s.ncols)[0]
    xh = xs + 1e-6 * ref.two_norm(xs) * u
    out["c2_grid32_verify"] = ref.verify_solution(s, xh, b, adam=cfg, restarts=1)
    out["c2_grid32_verify_inputs"] = {"x_seed": 17, "u_seed": 19, "rel_delta": 1e-6}
    # config 3 operator on a 16x16 grid
    h = configs.generate(configs.HYDROMECH, 16, 1)
    out["c3_grid16_projected_adam"] = _est(ref.projected_adam_explicit(h, cfg))
    # config 5 ensemble member shapes (n=4000, bandwidth 256)
    for idx in range(2):
        m = configs.ensemble_member(idx, 1, n=4000)
        c = ref.cond2(m, cfg, 4, 1e-14)
        out[f"c5_member{idx}_n4000_cond2_r4"] = {
            "kappa": c["kappa"], "operator_norm": _est(c["operator_norm"]),
            "inverse_norm": _est(c["inverse_norm"])}
    # config 2 sigma_max at full size (single run)
    a2 = configs.config(2)
    out["c2_projected_adam"] = _est(ref.projected_adam_explicit(a2, cfg))
    # single-SpMV checksums at full size for configs 1-3
    for k in (1, 2, 3):
        out[f"c{k}_spmv"] = spmv_checksums(ref, configs.config(k))
    _save("quick", out)


def column_scaled(a):
    """A D^-1 with D the column 2-norms (the paper's preconditioning, PAPER.md 'Condition
    Number and Preconditioning'); computed with numpy -- it is an input, not the path."""
    from paper_2409_11515_b200.sparse import SparseMatrix
    cn = np.zeros(a.ncols)
    np.add.at(cn, a.col_indices, a.values ** 2)
    cn = np.sqrt(cn)
    return SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices,
                        a.values / cn[a.col_indices])


def c5_scaled(ref):
    """Config-5 members have kappa >= 1/eps (per-column scales 10^U(-8,8)): the
    computed ||A^-1|| is then set by rounding, not by A, so kappa parity is asserted on
    the column-scaled members, where kappa is ~1e4."""
    out = {}
    cfg = configs.baseline_adam(1)
    for idx in range(2):
        m = column_scaled(configs.ensemble_member(idx, 1, n=4000))
        c = ref.cond2(m, cfg, 4, 1e-14)
        out[f"c5_member{idx}_n4000_colscaled_cond2_r4"] = {
            "kappa": c["kappa"], "operator_norm": _est(c["operator_norm"]),
            "inverse_norm": _est(c["inverse_norm"])}
    _save("c5_scaled", out)


def c3_sigma_max(ref):
    a = configs.config(3)
    t0 = time.time()
    e = ref.projected_adam_explicit(a, configs.baseline_adam(1))
    _save("c3_sigma_max", {"c3_projected_adam": _est(e), "seconds": time.time() - t0})


def c4_sigma_max(ref):
    a = configs.config(4)
    out = {"c4_spmv": spmv_checksums(ref, a)}
    t0 = time.time()
    e = ref.projected_adam_explicit(a, configs.baseline_adam(1))
    out["c4_projected_adam"] = _est(e)
    out["seconds"] = time.time() - t0
    _save("c4_sigma_max", out)


def c2_cond2(ref):
    a = configs.config(2)
    cfg = configs.baseline_adam(1)
    t0 = time.time()
    c = ref.cond2(a, cfg, 1, 1e-14)
    _save("c2_cond2", {"c2_cond2_r1": {"kappa": c["kappa"], "operator_norm": _est(c["operator_norm"]),
                                        "inverse_norm": _est(c["inverse_norm"])},
                       "seconds": time.time() - t0})


def c2_verify(ref):
    """verify_solution (error_bounds.hpp:166-217) on config 2 at full size: x* ~ U[-1,1)
    (seed 17), b = A x*, x^ = x* + 1e-6 ||x*|| u (u = random_unit_vector, seed 19), kappa
    estimated inside by cond2 with one restart per norm (the c2_cond2 run)."""
    a = configs.config(2)
    cfg = configs.baseline_adam(1)
    xs = ref.uniform_in(17, a.ncols, -1.0, 1.0)
    b = ref.matvec(a, xs)
    u = ref.random_unit_vectors(19, a.ncols)[0]
    xh = xs + 1e-6 * ref.two_norm(xs) * u
    t0 = time.time()
    rep = ref.verify_solution(a, xh, b, adam=cfg, restarts=1)
    _save("c2_verify", {"c2_verify_r1": rep, "inputs": {"x_seed": 17, "u_seed": 19,
                                                       "rel_delta": 1e-6},
                        "seconds": time.time() - t0})


def _c5_member_sigma_max(idx):
    ref = pyoracle.Oracle("ref")
    m = configs.ensemble_member(idx, 1)
    t0 = time.time()
    e = ref.estimate_norm_explicit(m, configs.baseline_adam(ref.mix_seed(1, 0x1000 + idx)), 4)
    return idx, _est(e), time.time() - t0


def c5_sigma_max(ref):
    """estimate_norm(ExplicitOracle, 4 restarts) of the first 8 full-size config-5 members
    (n = 100k); estimator seed mix_seed(1, 0x1000 + idx) (batch.member_seeds)."""
    from multiprocessing import Pool
    with Pool(4) as pool:
        res = pool.map(_c5_member_sigma_max, range(8))
    _save("c5_sigma_max", {f"c5_member{i}_estimate_norm_r4": {**e, "seconds": s}
                           for i, e, s in res})


def _c5_cond2(scaled):
    m = configs.ensemble_member(0, 1)
    if scaled:
        m = column_scaled(m)
    ref = pyoracle.Oracle("ref")
    cfg = configs.baseline_adam(ref.mix_seed(1, 0x1000))
    t0 = time.time()
    c = ref.cond2(m, cfg, 4, 1e-14)
    return {"kappa": c["kappa"], "operator_norm": _est(c["operator_norm"]),
            "inverse_norm": _est(c["inverse_norm"]), "seconds": time.time() - t0}


def c5_cond2(ref):
    """cond2 (4 restarts per norm) of full-size config-5 member 0, as generated and
    column-scaled (run_bench's per-matrix cond2, bench.hpp:430-442)."""
    from multiprocessing import Pool
    with Pool(2) as pool:
        raw, scaled = pool.map(_c5_cond2, [False, True])
    _save("c5_cond2", {"c5_member0_cond2_r4": raw, "c5_member0_colscaled_cond2_r4": scaled})


if __name__ == "__main__":
    job = sys.argv[1] if len(sys.argv) > 1 else "quick"
    ref = pyoracle.Oracle("ref")
    {"quick": quick, "c3_sigma_max": c3_sigma_max, "c4_sigma_max": c4_sigma_max,
     "c2_cond2": c2_cond2, "c5_scaled": c5_scaled, "c2_verify": c2_verify,
     "c5_sigma_max": c5_sigma_max, "c5_cond2": c5_cond2}[job](ref)
