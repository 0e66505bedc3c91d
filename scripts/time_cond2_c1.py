"""cond2 (condest.hpp:341-365) on config 1, warm: device (dense-block sweeps and,
with CK_LU_DENSE=0, the substitution sweeps) vs the compiled reference on one host core."""
import os
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_2409_11515_b200 as ck  # noqa: E402
import pyoracle  # noqa: E402
from paper_2409_11515_b200 import configs  # noqa: E402

a = configs.config(1)
cfg = configs.baseline_adam(1)
for mode in ("dense", "substitution"):
    if mode == "substitution":
        os.environ["CK_LU_DENSE"] = "0"
    ck.cond2(a, cfg)
    t0 = time.perf_counter()
    g = ck.cond2(a, cfg)
    t1 = time.perf_counter()
    f = ck.lu_factorize(a, 1e-14)
    c1 = configs.baseline_adam(ck.mix_seed(1, 0x1234))
    t2 = time.perf_counter()
    e = ck.inv_norm2(f, c1)
    t3 = time.perf_counter()
    print(f"{mode}: cond2 {t1 - t0:.3f} s kappa={g.kappa:.12e} inv={g.inverse_norm.value:.12e}; one inverse run "
          f"{t3 - t2:.3f} s = {1e3 * (t3 - t2) / max(e.iterations, 1):.3f} ms/iteration, dense_info={f.dense_info()}",
          flush=True)
os.environ.pop("CK_LU_DENSE", None)
if len(sys.argv) > 1 and sys.argv[1] == "ref":
    ref = pyoracle.Oracle("ref" if pyoracle.available("ref") else "port")
    t2 = time.perf_counter()
    r = ref.cond2(a, cfg)
    t3 = time.perf_counter()
    print(f"reference (1 host core): cond2 {t3 - t2:.3f} s kappa={(r['kappa'] if isinstance(r, dict) else r.kappa):.12e}")
