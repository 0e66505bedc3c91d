"""Config-5 sigma_min throughput: a wave of full-size ensemble members, one
CTA per member, R = 4 restarts each (the factorisations run concurrently)."""
import sys, time
sys.path.insert(0, ".")
from paper_2409_11515_b200 import batch, configs

for S in [int(a) for a in sys.argv[1:]] or [16, 64]:
    mem = [configs.ensemble_member(g, 1) for g in range(S)]
    t0 = time.perf_counter()
    facs = batch.lu_factorize_many(mem, 1e-14, threads=16)
    tf = time.perf_counter() - t0
    cfg = configs.baseline_adam(3, max_iter=100000)
    s = batch.InverseBatchSession(facs, cfg, list(range(1, 4 * S + 1)))
    s.run(4)
    steps = 10
    ms, _, _ = s.time(steps, 1)
    it = S * 4 * steps / (ms / 1e3)
    print(f"S={S}: factor {tf:.2f}s ({tf / S * 1e3:.0f} ms/member), step {ms / steps:.2f} ms -> "
          f"{it:.0f} run-iterations/s", flush=True)
    del s, facs
