"""sigma_min step time vs members sharing one factorisation (one CTA each),
config 1 (restarts as members, as estimate_norm/cond2 run them)."""
import sys

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import batch, configs, inverse  # noqa: E402

a = configs.config(1)
f = ck.lu_factorize(a, 1e-14)
steps = 100
for S in (1, 2, 3, 4, 8):
    s = batch.InverseBatchSession([f] * S, configs.baseline_adam(3, max_iter=100000), list(range(3, 3 + S)))
    s.run(4)
    ms, _, _ = s.time(steps, 1)
    print(f"S={S}: {ms / steps:.3f} ms/step", flush=True)
for R in (1, 2, 3, 4):
    s = inverse.InverseSession(ck.InverseOracle(f), configs.baseline_adam(3, max_iter=100000), list(range(3, 3 + R)))
    s.run(4)
    ms, _, _ = s.time(steps, 1)
    print(f"R={R} columns: {ms / steps:.3f} ms/step", flush=True)
