"""Cluster-split sweeps vs the single-CTA sweeps on the same factorisation:
the solves and a short sigma_min run must agree to rounding (CK_LU_CLUSTER
selects the split per process, so the two runs are separate processes)."""
import json
import os
import subprocess
import sys

code = r'''
import sys, json, time
sys.path.insert(0, ".")
import numpy as np
import paper_2409_11515_b200 as ck
from paper_2409_11515_b200 import configs, inverse
name = sys.argv[1]
a = {"c1": lambda: configs.config(1), "c2": lambda: configs.config(2),
     "c5m0": lambda: configs.ensemble_member(0, 1)}[name]()
f = ck.lu_factorize(a, 1e-14)
cfg = configs.baseline_adam(3, max_iter=int(sys.argv[2]))
s = inverse.InverseSession(ck.InverseOracle(f), cfg, [3])
t0 = time.perf_counter()
s.run()
t1 = time.perf_counter()
e = s.result(0)
print(json.dumps({"value": e.value, "its": e.iterations, "ms_per_it": (t1 - t0) / e.iterations * 1e3,
                  "w0": float(e.witness[0])}))
'''
for name, its in [("c1", 200), ("c5m0", 40), ("c2", 20)]:
    out = {}
    for cl in os.environ.get("CK_CL_LIST", "1 8").split():
        env = dict(os.environ, CK_LU_CLUSTER=cl)
        if cl == "auto":
            env.pop("CK_LU_CLUSTER")
        r = subprocess.run([sys.executable, "-c", code, name, str(its)], capture_output=True, text=True,
                           env=env, timeout=900)
        if r.returncode:
            print(name, cl, "FAILED", r.stderr[-500:], flush=True)
            continue
        out[cl] = json.loads(r.stdout.strip().splitlines()[-1])
    if "1" in out:
        for k, v in out.items():
            rel = abs(v["value"] - out["1"]["value"]) / out["1"]["value"]
            print(f"{name}: cluster {k}: {v['ms_per_it']:.3f} ms/it, value rel diff vs one CTA {rel:.2e}, "
                  f"its {v['its']}", flush=True)
