"""Phase breakdown of the e2e call bench.py times (norm2 from pinned host CSR
on config 4); run with CK_TRACE=1 for the native phase marks. The call is made
twice: the second pass (warm modules and allocator) is what bench.py's e2e sees."""
import gc
import sys
import time

sys.path.insert(0, ".")
import paper_2409_11515_b200 as ck  # noqa: E402
from paper_2409_11515_b200 import _lib, configs  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
c = configs.CONFIGS[cfg_id]
a = configs.generate(c["kind"], c["grid"], 1, c["param"])
for arr in (a.row_offsets, a.col_indices, a.values):
    _lib.check(_lib.load().ck_host_register(arr.ctypes.data, arr.nbytes), "ck_host_register")
noprefetch = "noprefetch" in sys.argv
for p in ("cold", "warm", "warm2"):
    a2 = ck.SparseMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, a.values, validate=False)
    cfg = configs.baseline_adam(1, max_iter=iters)
    print(f"--- {p} pass", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    if not noprefetch:
        _lib.check(_lib.load().ck_start_vector_prefetch(cfg.seed, a2.ncols), "prefetch")  # norm2's order
    dev = a2.device()
    t1 = time.perf_counter()
    s = ck.Session(ck.ExplicitOracle(a2), cfg, [cfg.seed])
    t2 = time.perf_counter()
    s.run()
    t3 = time.perf_counter()
    est = s.result(0)
    t4 = time.perf_counter()
    s.close()
    del s, dev, a2
    gc.collect()
    t5 = time.perf_counter()
    print(f"{p}: upload+build {t1 - t0:.3f} s, session {t2 - t1:.3f} s, loop {t3 - t2:.3f} s "
          f"({est.iterations} its, {(t3 - t2) / est.iterations * 1e3:.3f} ms/it), result {t4 - t3:.3f} s, "
          f"release {t5 - t4:.3f} s, total {t5 - t0:.3f} s -> {est.iterations / (t5 - t0):.1f} it/s", flush=True)
