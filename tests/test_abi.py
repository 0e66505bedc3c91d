"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/*.h declares, and its host-side functions (RNG mirror, scalar
error bounds) agree with the reference oracle bit for bit."""
import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import _lib, error_bounds as eb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    out = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            text = open(os.path.join(ROOT, "include", h)).read()
            out |= set(re.findall(r"\b(ck_[a-z0-9_]+)\s*\(", text))
    return out


def test_every_declared_symbol_is_exported():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) > 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r" T (ck_\w+)", nm))
    assert syms <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_abi_version_and_defaults():
    lib = _lib.load()
    assert lib.ck_abi_version() == 1
    c = _lib.AdamCfg()
    lib.ck_adam_default(C.byref(c))
    d = ck.AdamConfig()
    for f, _ in _lib.AdamCfg._fields_:
        assert getattr(c, f) == getattr(d, f)


def test_rng_mirror_bitwise(port):
    assert ck.mix_seed(1, 0x1234) == port.mix_seed(1, 0x1234)
    assert np.array_equal(ck.random_unit_vectors(11, 333, 5), port.random_unit_vectors(11, 333, 5))
    # the threaded Box-Muller path (n >= 2^18)
    assert np.array_equal(ck.random_unit_vector(300_000, 4), port.random_unit_vectors(4, 300_000)[0])
    # several pipeline blocks (2^18 pairs each) and a ragged last block
    assert np.array_equal(ck.random_unit_vectors(9, 600_001, 2), port.random_unit_vectors(9, 600_001, 2))


def test_bounds_match_oracle(port):
    rng = np.random.default_rng(0)
    for _ in range(200):
        rn, bn, an, xn = 10.0 ** rng.uniform(-12, 2, 4)
        k = 10.0 ** rng.uniform(0, 17)
        assert eb.loose_bounds(rn, bn, k) == eb.Bounds(*port.loose_bounds(rn, bn, k))
        assert eb.tight_bounds(rn, an, xn, k) == eb.Bounds(*port.tight_bounds(rn, an, xn, k))
        assert eb.singularity_bound(k) == port.singularity_bound(k)
        e = 10.0 ** rng.uniform(-12, 0.5)
        assert eb.propagate_bound(e) == port.propagate_bound(e)
    with pytest.raises(ck.ZeroRHS):
        eb.loose_bounds(0.1, 0.0, 2.0)
    with pytest.raises(ck.ZeroSolution):
        eb.tight_bounds(0.1, 1.0, 0.0, 2.0)
    with pytest.raises(ValueError):
        eb.loose_bounds(0.1, 1.0, 0.5)
    with pytest.raises(ValueError):
        eb.propagate_bound(-1e-30)
    assert math.isinf(eb.singularity_bound(2.0 ** 53))


def test_sparse_matrix_validation():
    # test_sparse.cpp:36-41
    with pytest.raises(ck.DimensionMismatch):
        ck.SparseMatrix(1, 1, [0, 2], [0], [1.0])
    with pytest.raises(ck.DimensionMismatch):
        ck.SparseMatrix(1, 2, [0, 2], [1, 0], [1.0, 2.0])
    with pytest.raises(ck.DimensionMismatch):
        ck.SparseMatrix(1, 1, [0, 1], [1], [1.0])
    with pytest.raises(ck.DimensionMismatch):
        ck.SparseMatrix(1, 1, [0, 1], [0], [float("nan")])
    a = ck.SparseMatrix.from_triplets(2, 2, [(0, 1, 2.0), (0, 0, 1.0), (0, 1, 3.0)])
    assert a.nnz == 2 and a.coeff(0, 1) == 5.0 and a.coeff(1, 0) == 0.0
    with pytest.raises(ck.DimensionMismatch):
        ck.SparseMatrix.from_triplets(2, 2, [(2, 0, 1.0)])


def test_no_silent_cpu_path_without_gpu():
    n = C.c_int32()
    _lib.check(_lib.load().ck_device_count(C.byref(n)))
    if n.value > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(ck.DeviceUnavailable):
        ck.norm2(ck.SparseMatrix.identity(4))
    with pytest.raises(ck.DeviceUnavailable):
        ck.matvec(ck.SparseMatrix.identity(4), np.ones(4))


def _build_dropin(tmp_path, with_reference):
    exe = tmp_path / ("dropin_ref" if with_reference else "dropin")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "dropin_demo.cpp"),
           "-L", os.path.dirname(_lib.LIB_PATH), "-lcondkit_b200",
           "-Wl,-rpath," + os.path.dirname(_lib.LIB_PATH), "-o", str(exe)]
    if with_reference:
        cmd[3:3] = ["-I", "/root/reference/proj/include", "-DWITH_REFERENCE_TYPES"]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_cpp_dropin_header_compiles_against_reference_types(tmp_path):
    # the reference's own condkit::SparseMatrix flows into condkit_b200::cond2 unchanged
    if not os.path.isdir("/root/reference/proj/include/condkit"):
        pytest.skip("reference headers not present on this machine")
    assert _build_dropin(tmp_path, True).exists()


def test_cpp_dropin_header_compiles_standalone(tmp_path):
    assert _build_dropin(tmp_path, False).exists()


def test_reference_demos_build_against_b200_headers():
    # proj/include/condkit (B200 condest.hpp / lu.hpp / error_bounds.hpp) shadows the
    # reference's headers: the reference's demos and its unit-test call sites compile
    # unchanged (-Wall -Wextra); the GPU half runs them (tests/test_gpu_dropin.py)
    if not os.path.isdir("/root/reference/proj/include/condkit"):
        pytest.skip("reference headers not present on this machine")
    from paper_2409_11515_b200 import build
    exes = build.build_dropin()
    for name in ("condest_checks", "condition_estimate", "residual_vs_error"):
        assert os.path.join(build.DROPIN, name) in exes
    for d in build.DEMOS:
        assert os.path.getsize(os.path.join(ROOT, "tests", "golden", f"dropin_{d}.txt")) > 0
