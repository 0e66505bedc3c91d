"""The C++ drop-in header (include/condkit_b200.hpp) driving the device."""
import os
import subprocess

import numpy as np
import pytest

import paper_2409_11515_b200 as ck
from test_abi import _build_dropin

pytestmark = pytest.mark.gpu


def _grid_matrix(g):
    t = []
    for r in range(g):
        for c in range(g):
            i = r * g + c
            t.append((i, i, 4.0 + 0.01 * (i % 7)))
            if r > 0:
                t.append((i, i - g, -1.0))
            if r + 1 < g:
                t.append((i, i + g, -1.0))
            if c > 0:
                t.append((i, i - 1, -1.0))
            if c + 1 < g:
                t.append((i, i + 1, -1.0))
    return ck.SparseMatrix.from_triplets(g * g, g * g, t)


def test_cpp_dropin_runs_and_matches_python(tmp_path):
    exe = _build_dropin(tmp_path, False)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    vals = dict(zip(out[0::2], out[1::2]))
    r = ck.cond2(_grid_matrix(12))
    assert float(vals["kappa"]) == r.kappa  # same device path, same bits
    assert float(vals["sigma_max"]) == r.operator_norm.value
