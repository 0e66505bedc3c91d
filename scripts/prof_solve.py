"""Runs the standalone band solves (k_lu_solve) on a config's factors -- the
target of the ncu captures of the sigma_min sweeps."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
a = configs.config(1) if which == "c1" else configs.ensemble_member(0, 1) if which == "c5m0" else configs.config(2)
f = ck.lu_factorize(a, 1e-14)
b = np.random.default_rng(1).standard_normal(a.nrows)
for _ in range(3):
    x = f.solve(b)
    y = f.transpose_solve(b)
print(which, "ok", float(np.linalg.norm(x)), float(np.linalg.norm(y)))
