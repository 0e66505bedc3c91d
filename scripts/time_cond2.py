"""End-to-end cond2 (condest.hpp:341-365) on the device vs the compiled
reference on one host core, warm (after a first call): config 1, and the
factorisation alone on configs 1, 2 and a config-5 member."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_2409_11515_b200 as ck  # noqa: E402
import pyoracle  # noqa: E402
from paper_2409_11515_b200 import configs  # noqa: E402

for name, a in [("c1", configs.config(1)), ("c5m0", configs.ensemble_member(0, 1)), ("c2", configs.config(2))]:
    a.device()
    ck.lu_factorize(a, 1e-14)  # warm: module loading, allocations
    t0 = time.perf_counter()
    f = ck.lu_factorize(a, 1e-14)
    t1 = time.perf_counter()
    print(f"{name}: lu_factorize (warm) {t1 - t0:.3f} s, n={f.n} kl={f.kl} ku={f.ku}", flush=True)

a = configs.config(1)
cfg = configs.baseline_adam(1)
ck.cond2(a, cfg)
t0 = time.perf_counter()
g = ck.cond2(a, cfg)
t1 = time.perf_counter()
ref = pyoracle.Oracle("ref" if pyoracle.available("ref") else "port")
t2 = time.perf_counter()
r = ref.cond2(a, cfg)
t3 = time.perf_counter()
print(f"c1 cond2 (3 restarts, 2000 its): device {t1 - t0:.3f} s kappa={g.kappa:.9e}; "
      f"reference 1 core {t3 - t2:.3f} s kappa={r['kappa']:.9e}", flush=True)

# phases of the device cond2 on config 1 (warm)
t0 = time.perf_counter()
e = ck.estimate_norm(ck.ExplicitOracle(a), cfg, 3)
t1 = time.perf_counter()
f = ck.lu_factorize(a, 1e-14)
t2 = time.perf_counter()
ci = configs.baseline_adam(ck.mix_seed(1, 0x1234))
ei = ck.estimate_norm(ck.InverseOracle(f), ci, 3)
t3 = time.perf_counter()
print(f"c1 cond2 phases: sigma_max {t1 - t0:.3f} s ({e.iterations} its), LU {t2 - t1:.3f} s, "
      f"sigma_min {t3 - t2:.3f} s ({ei.iterations} its)", flush=True)
