"""Small runs of every device path for compute-sanitizer (memcheck / racecheck /
synccheck): the sigma_max sweeps (R = 1, 2), the batched ensemble (window and
global gathers), the band LU (panel + trailing update + CSR export + dense
blocks), the inverse sweeps on 8-CTA clusters (kl + ku >= 256), on one CTA and
as dense-block sweeps, and a 4-rank in-process partition."""
import sys

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import batch, configs  # noqa: E402

cfg = configs.baseline_adam(1, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 30)
lap = configs.generate(configs.LAPLACIAN, 32, 1)
print("norm2", ck.norm2(lap, cfg).value)
print("estimate_norm R=2", ck.estimate_norm(ck.ExplicitOracle(lap), cfg, 2).value)
mem = [configs.ensemble_member(i, 1, n=1200, bw=64) for i in range(3)]
print("batch", [e.value for e in batch.estimate_norm_batch(mem, cfg, 2)])
band = configs.ensemble_member(3, 1, n=1500, bw=150)  # kl + ku ~ 300: cluster sweeps
f = ck.lu_factorize(band, 1e-14)
print("lu", f.kl, f.ku, f.export_csr()[0].nnz)
print("inv_norm2 (cluster)", ck.inv_norm2(f, cfg).value)
g = ck.lu_factorize(lap, 1e-14)
print("inv_norm2 (dense-block sweeps)", g.dense_info(), ck.inv_norm2(g, cfg).value)
import os  # noqa: E402
os.environ["CK_LU_DENSE"] = "0"
g = ck.lu_factorize(lap, 1e-14)
print("inv_norm2 (substitution sweeps, one CTA)", ck.inv_norm2(g, cfg).value)
del os.environ["CK_LU_DENSE"]
os.environ["CK_NO_WINDOW"] = "1"
print("batch (global gathers)", [e.value for e in batch.estimate_norm_batch(mem, cfg, 2)])
del os.environ["CK_NO_WINDOW"]
from paper_2409_11515_b200 import dist  # noqa: E402
print("partition, 4 ranks in process", [e.value for e in dist.projected_adam_partitioned(lap, 4, cfg, seeds=[1, 2])])
