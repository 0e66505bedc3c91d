"""Per-phase cycles of the band sweeps inside the inverse Projected-Adam step
(profiling build, CK_LIB=...libcondkit_b200_prof.so), single-CTA or cluster
(CK_LU_CLUSTER). Counts are the leader CTA's thread 0; several restarts/members
add up, so run one system."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("CK_LIB", os.path.abspath("paper_2409_11515_b200/libcondkit_b200_prof.so"))
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import _lib, configs, inverse  # noqa: E402

lib = _lib.load()
fn = lib.ck_debug_sweep_prof_inv
buf = (C.c_ulonglong * 32)()
names = ["L fwd", "U bwd", "U^T fwd", "L^T bwd"]
phases = ["phase1", "bar1", "phase2", "bar2"]
for which in sys.argv[1:] or ["c2"]:
    a = {"c1": lambda: configs.config(1), "c5m0": lambda: configs.ensemble_member(0, 1),
         "c2": lambda: configs.config(2)}[which]()
    f = ck.lu_factorize(a, 1e-14)
    s = inverse.InverseSession(ck.InverseOracle(f), configs.baseline_adam(3, max_iter=100000), [3])
    s.run(2)
    fn(buf, 1)
    steps = 4
    s.run(steps)
    fn(buf, 1)
    nblk = (a.nrows + 31) // 32
    print(f"{which}: n={a.nrows} kl={f.kl} ku={f.ku} cluster={os.environ.get('CK_LU_CLUSTER', 'auto')}  "
          f"cycles per block (leader thread 0)")
    for k in range(4):
        v = [buf[8 * k + 2 * p] / (steps * nblk) for p in range(2)] + [buf[8 * k + 4 + p] / (steps * nblk) for p in range(2)]
        print(f"  {names[k]:8s} " + "  ".join(f"{ph} {x:7.0f}" for ph, x in zip(phases, v)) + f"  total {sum(v):7.0f}")
