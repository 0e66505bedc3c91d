"""A/B of the sigma_min iteration across library builds (CK_LIB per run):
ms per inverse iteration on config 1, a config-5 member and config 2."""
import os
import subprocess
import sys

code = r'''
import sys, time
sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs, inverse
out = []
for name, a in [("c1", configs.config(1)), ("c5m0", configs.ensemble_member(0, 1)), ("c2", configs.config(2))]:
    f = ck.lu_factorize(a, 1e-14)
    cfg = configs.baseline_adam(3, max_iter=100000)
    s = inverse.InverseSession(ck.InverseOracle(f), cfg, [3])
    s.run(4)
    steps = 40 if name != "c2" else 10
    ms, _, _ = s.time(steps, 1)
    out.append(f"{name} {ms / steps:.3f}")
print("  ".join(out))
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        env = dict(os.environ, CK_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
        print(f"{lib:14s} {r.stdout.strip()} {r.stderr.strip()[-200:] if r.returncode else ''}", flush=True)
