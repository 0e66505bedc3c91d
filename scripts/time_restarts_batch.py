"""Config 5 ensemble: per-step time of the packed sigma_max sweeps vs the
restart columns per sweep (the 4 restarts as 1, 2 or 4 columns)."""
import sys

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import batch, configs  # noqa: E402

nm = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = configs.CONFIGS[5]
mem = [configs.ensemble_member(i, 1, n=c["grid"], bw=c["param"]) for i in range(nm)]
packed = batch.pack_block_diagonal(mem)
ms_seeds = batch.member_seeds(nm)
steps = 50
for R in (1, 2, 4):
    seeds = [ms_seeds[i] if r == 0 else ck.mix_seed(ms_seeds[i], r) for i in range(nm) for r in range(R)]
    s = batch.BatchSession(packed, configs.baseline_adam(1, max_iter=3 * steps + 20), seeds)
    s.run(5)
    tot, ap, tr = s.time(steps, mode=0)
    tot1, _, _ = s.time(steps, mode=1)
    s.close()
    print(f"config 5 x{nm}, R={R}: {tot1 / steps:.3f} ms/step (graph; apply {ap / steps:.3f}, "
          f"transpose {tr / steps:.3f}); 4 restarts cost {4 / R * tot1 / steps:.3f} ms/step", flush=True)
