"""Per-phase cycle counts of the four band sweeps (profiling build:
`python -m paper_2409_11515_b200.build --prof`, then CK_LIB=... this)."""
import ctypes as C, os, sys
sys.path.insert(0, ".")
os.environ.setdefault("CK_LIB", os.path.abspath("paper_2409_11515_b200/libcondkit_b200_prof.so"))
import numpy as np
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs, _lib

lib = _lib.load()
buf = (C.c_ulonglong * 32)()
names = ["L fwd", "U bwd", "U^T fwd", "L^T bwd"]
phases = ["phase1", "bar1", "phase2", "bar2"]
for which in sys.argv[1:] or ["c1"]:
    a = {"c1": lambda: configs.config(1), "c5m0": lambda: configs.ensemble_member(0, 1),
         "c2": lambda: configs.config(2)}[which]()
    f = ck.lu_factorize(a, 1e-14)
    b = np.random.default_rng(1).standard_normal(a.nrows)
    f.solve(b); f.transpose_solve(b)
    lib.ck_debug_sweep_prof(buf, 1)
    reps = 5
    for _ in range(reps):
        f.solve(b); f.transpose_solve(b)
    lib.ck_debug_sweep_prof(buf, 1)
    nblk = (a.nrows + 31) // 32
    print(f"{which}: n={a.nrows} kl={f.kl} ku={f.ku}  cycles per block (thread 0)")
    for s in range(4):
        v = [buf[8 * s + 2 * p] / (reps * nblk) for p in range(2)] + [buf[8 * s + 4 + p] / (reps * nblk) for p in range(2)]
        print(f"  {names[s]:8s} " + "  ".join(f"{ph} {x:7.0f}" for ph, x in zip(phases, v)) + f"  total {sum(v):7.0f}")
