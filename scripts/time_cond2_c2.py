"""cond2 end to end on config 2 (n = 196,608, kl = ku = 769): sigma_max by
estimate_norm (3 restarts), the device band LU, sigma_min (3 restarts on
8-CTA clusters, side by side), 2000 iterations each (BASELINE settings)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import configs  # noqa: E402

a = configs.config(2)
cfg = configs.baseline_adam(1)
a.device()
t0 = time.perf_counter()
e = ck.estimate_norm(ck.ExplicitOracle(a), cfg, 3)
t1 = time.perf_counter()
f = ck.lu_factorize(a, 1e-14)
t2 = time.perf_counter()
ci = configs.baseline_adam(ck.mix_seed(1, 0x1234))
ei = ck.estimate_norm(ck.InverseOracle(f), ci, 3)
t3 = time.perf_counter()
print(f"c2 cond2: sigma_max {e.value:.9e} ({t1 - t0:.2f} s), LU {t2 - t1:.2f} s (kl={f.kl} ku={f.ku}), "
      f"||A^-1|| {ei.value:.9e} ({t3 - t2:.1f} s, {ei.iterations} its), kappa {e.value * ei.value:.6e}, "
      f"total {t3 - t0:.1f} s", flush=True)
