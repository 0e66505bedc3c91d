"""Warm lu_factorize timings (config 1, a config-5 member, config 2) for A/B runs of the
factorisation kernels; `--only c5m0` limits the set (ncu captures)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import configs  # noqa: E402

only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
cases = [("c1", lambda: configs.config(1)), ("c5m0", lambda: configs.ensemble_member(0, 1)),
         ("c2", lambda: configs.config(2))]
for name, make in cases:
    if only and name != only:
        continue
    a = make()
    a.device()
    if not only:
        ck.lu_factorize(a, 1e-14)  # warm: module loading, allocations
    t0 = time.perf_counter()
    f = ck.lu_factorize(a, 1e-14)
    t1 = time.perf_counter()
    print(f"{name}: lu_factorize {t1 - t0:.3f} s, n={f.n} kl={f.kl} ku={f.ku}", flush=True)
