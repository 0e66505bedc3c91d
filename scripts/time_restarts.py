"""Per-iteration time of the fused sweeps vs the restart-column count R
(estimate_norm / cond2 run R restarts as columns of one sweep)."""
import sys

import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = configs.CONFIGS[cfg_id]
a = configs.generate(c["kind"], c["grid"], 1, c["param"])
steps = 100
for R in (1, 2, 3, 4):
    cfg = configs.baseline_adam(1, max_iter=3 * steps + 20)
    s = ck.Session(ck.ExplicitOracle(a), cfg, [ck.mix_seed(1, r) for r in range(R)])
    s.run(5)
    tot, ap, tr = s.time(steps, mode=0)
    tot1, _, _ = s.time(steps, mode=1)
    s.close()
    print(f"config {cfg_id} R={R}: {tot1 / steps:.4f} ms/step (graph), apply {ap / steps:.4f} "
          f"transpose {tr / steps:.4f} ms; per restart-iteration {tot1 / steps / R:.4f} ms", flush=True)
