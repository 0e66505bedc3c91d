"""Per-iteration cost of the row-block partition's rank-local work:
all P ranks of config 4 (or --grid G of config 3's operator) driven in one process on
one device -- P ranks' sweeps back to back plus the pack / combine kernels and device
copies that stand in for the NCCL exchange -- against the single-device loop.
usage: python scripts/time_partition.py [P=8] [grid=2048] [steps=50]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import configs, dist  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
a = configs.generate(3, grid)
cfg = configs.baseline_adam(1, max_iter=10**7)
one = ck.Session(ck.ExplicitOracle(a), cfg, [1])
one.run(5)
t1 = one.time(steps, mode=1)[0] / steps
one.close()
t0 = time.perf_counter()
parts = dist.build_partition(a, P)
tb = time.perf_counter() - t0
halo_x = [int(p.lists["xs_off"][-1]) for p in parts]
halo_y = [int(p.lists["ys_off"][-1]) for p in parts]
s = dist.PartitionedSession(parts, cfg, [1])
s.run(5)
tp = s.time(steps) / steps
s.free()
print(f"grid {grid}: n={a.nrows} nnz={a.nnz}; single device {t1:.4f} ms/iteration")
print(f"P={P} ranks in one process: {tp:.4f} ms/iteration for all ranks = {tp / P:.4f} ms per rank-iteration "
      f"(ideal {t1 / P:.4f}); rank-local overhead {1e3 * (tp - t1) / P:.1f} us per rank-iteration "
      f"(2 packs + 2 combines + copies, sub-wave sweeps)")
print(f"halo entries per rank per iteration: x side {max(halo_x)} x 16 B, y side {max(halo_y)} x 8 B "
      f"= {(16 * max(halo_x) + 8 * max(halo_y)) / 1e3:.1f} kB; partials {8 * 10} B to every peer; "
      f"partition build (host) {tb:.1f} s")
