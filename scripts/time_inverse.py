"""Times the sigma_min (inverse) iteration and the factorisation on configs 1, 2 and a config-5 member."""
import sys, time
sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs, inverse

for name, a in [("c1", configs.config(1)), ("c5m0", configs.ensemble_member(0, 1)),
                ("c2", configs.config(2))]:
    t0 = time.perf_counter(); f = ck.lu_factorize(a, 1e-14); tf = time.perf_counter() - t0
    cfg = configs.baseline_adam(3, max_iter=100000)
    s = inverse.InverseSession(ck.InverseOracle(f), cfg, [3])
    s.run(4)
    steps = 40 if name != "c2" else 10
    ms, _, _ = s.time(steps, 1)
    print(f"{name}: n={f.n} kl={f.kl} ku={f.ku} factor {tf:.3f}s  inverse iteration {ms/steps:.3f} ms"
          f"  (2000 its: {2 * ms / steps:.1f} s)", flush=True)
