"""A/B of the restart-column sweeps across library builds (CK_LIB per run)."""
import os
import subprocess
import sys

for lib in sys.argv[1:]:
    env = dict(os.environ, CK_LIB=os.path.abspath(lib), PYTHONPATH=os.getcwd())
    for script in ("scripts/time_restarts.py", "scripts/time_restarts_batch.py"):
        r = subprocess.run([sys.executable, script], capture_output=True, text=True, env=env)
        for line in r.stdout.strip().splitlines():
            print(f"{lib:10s} {line}", flush=True)
        if r.returncode:
            print(lib, r.stderr[-300:])
