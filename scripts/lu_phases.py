"""Panel-kernel phase cycles of lu_factorize (profiling build: python -m
paper_2409_11515_b200.build --prof, then CK_LIB=.../libcondkit_b200_prof.so)."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import _lib, configs  # noqa: E402

lib = _lib.load()
buf = (C.c_ulonglong * 32)()
names = {2: "search", 3: "reduce+pivot", 6: "swap", 7: "order keys", 10: "rank+divide",
         11: "panel update"}
for name, a in [("c5m0", configs.ensemble_member(0, 1)), ("c2", configs.config(2))]:
    a.device()
    lib.ck_debug_sweep_prof(buf, 1)
    t0 = time.perf_counter()
    f = ck.lu_factorize(a, 1e-14)
    dt = time.perf_counter() - t0
    lib.ck_debug_sweep_prof(buf, 1)
    tot = sum(buf[k] for k in names)
    print(f"{name}: {dt:.3f} s, panel cycles {tot / 1e9:.2f} G ({tot / 1.9e9:.2f} s at 1.9 GHz)")
    for k, nm in names.items():
        print(f"   {nm:14s} {buf[k] / max(tot, 1) * 100:5.1f}%  {buf[k] / f.n:9.0f} cyc/column")
