"""A/B of the config-4 loop across library builds (CK_LIB): graph-timed
iterations/s and the per-kernel split, same box, interleaved runs."""
import json, os, subprocess, sys
libs = sys.argv[1:]
for rep in range(2):
    for lib in libs:
        env = dict(os.environ)
        if lib != "default":
            env["CK_LIB"] = os.path.abspath(lib)
        out = subprocess.run([sys.executable, "bench.py", "--no-e2e", "--no-cpu", "--steps", "200",
                              "--warmup", "5"], capture_output=True, text=True, env=env).stdout
        d = json.loads(out.strip().splitlines()[-1])
        k = d["kernels"]
        print(f"{lib:16s} {d['value']:7.1f} it/s  apply {k['apply']['ms_avg']:.4f} ms  "
              f"transpose {k['transpose']['ms_avg']:.4f} ms  sm {d['clocks']['sm_mhz'] if d['clocks'] else None}",
              flush=True)
