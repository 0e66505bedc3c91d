"""Config-1 inverse iteration (device time from CUDA-graph chunks): dense-block sweeps vs
the substitution sweeps (CK_LU_DENSE=0), 1 and 3 systems side by side."""
import os
import sys

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import batch, configs, inverse  # noqa: E402

a = configs.config(1)
cfg = configs.baseline_adam(3, max_iter=10**7)
for mode in ("dense", "substitution"):
    if mode == "substitution":
        os.environ["CK_LU_DENSE"] = "0"
    f = ck.lu_factorize(a, 1e-14)
    s = inverse.InverseSession(ck.InverseOracle(f), cfg, [3])
    s.run(64)
    one = [s.time(640, 1)[0] / 640 for _ in range(3)]
    s3 = batch.InverseBatchSession([f, f, f], cfg, [3, 4, 5])
    s3.run(64)
    three = [s3.time(640, 1)[0] / 640 for _ in range(3)]
    print(f"{mode}: dense_info={f.dense_info()} one system {min(one):.4f} ms/iteration "
          f"(runs {['%.4f' % t for t in one]}); three systems side by side {min(three):.4f} ms/step", flush=True)
