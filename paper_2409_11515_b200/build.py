"""In-tree build of the native library (sm_100a only).

``python -m paper_2409_11515_b200.build`` compiles every CUDA/C++ source under
csrc/ into ``paper_2409_11515_b200/libcondkit_b200.so`` with nvcc. The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libcondkit_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.h")) +
                  glob.glob(os.path.join(PKG, "csrc", "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, prof: bool = False) -> str:
    """prof=True builds the phase-timing variant (-DCK_SWEEP_PROF) next to
    the library as libcondkit_b200_prof.so (load it with CK_LIB=...).

    Each translation unit compiles to its own object in parallel (build/),
    then nvcc links the shared library."""
    out = LIB.replace(".so", "_prof.so") if prof else LIB
    if not prof and not force and not needs_build():
        return LIB
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
             "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc")]
    if prof:
        flags.insert(0, "-DCK_SWEEP_PROF")
    flags = os.environ.get("CK_NVCC_FLAGS", "").split() + flags  # A/B builds
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    objdir = os.path.join(ROOT, "build", "prof" if prof else "lib")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC] + flags + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {failed}")
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-o", out + ".tmp"] + objs + ["-lpthread"], check=True)
    os.replace(out + ".tmp", out)
    if not prof:
        build_cli()
        build_dropin()
    return out


CLI = os.path.join(ROOT, "tools", "condkit_b200_cli")


def build_cli() -> str:
    """tools/condkit_b200_cli: the cond/norm/verify/convert front end (C++,
    over include/condkit_b200.hpp and the in-tree library)."""
    src = os.path.join(ROOT, "tools", "condkit_b200_cli.cpp")
    cmd = ["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), src, "-o",
           CLI + ".tmp", "-L", PKG, "-lcondkit_b200", f"-Wl,-rpath,{PKG}",
           "-Wl,-rpath,$ORIGIN/../paper_2409_11515_b200"]
    subprocess.run(cmd, check=True)
    os.replace(CLI + ".tmp", CLI)
    return CLI


REF_INC = "/root/reference/proj/include"
REF_DEMO = "/root/reference/proj/demo"
DROPIN = os.path.join(ROOT, "build", "dropin")
DEMOS = ("condition_estimate", "residual_vs_error")


def build_dropin() -> list:
    """The reference's own call sites against the B200 headers of proj/include/condkit
    (they shadow the reference's condest.hpp, lu.hpp, error_bounds.hpp), built into
    build/dropin/ where the reference headers exist (this container; the binaries travel
    to the GPU box with the snapshot, which has no reference tree):
      condest_checks      tests/cpp/dropin_condest_checks.cpp
      <demo>              the reference's demo/<demo>.cpp, unchanged
    and, as the parity anchor, the same demos against the reference alone (ref_<demo>),
    whose output is recorded in tests/golden/dropin_<demo>.txt."""
    if not os.path.isdir(os.path.join(REF_INC, "condkit")):
        return []
    os.makedirs(DROPIN, exist_ok=True)
    ours = ["-I", os.path.join(ROOT, "proj", "include"), "-I", os.path.join(ROOT, "include"),
            "-I", REF_INC]
    link = ["-L", PKG, "-lcondkit_b200", "-Wl,-rpath,$ORIGIN/../../paper_2409_11515_b200",
            "-lpthread"]
    jobs = [(os.path.join(ROOT, "tests", "cpp", "dropin_condest_checks.cpp"), "condest_checks",
             ours, link)]
    for d in DEMOS:
        src = os.path.join(REF_DEMO, d + ".cpp")
        jobs.append((src, d, ours, link))
        jobs.append((src, "ref_" + d, ["-I", REF_INC], ["-lpthread"]))
    procs = []
    for src, name, inc, lk in jobs:
        exe = os.path.join(DROPIN, name)
        cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra"] + inc + [src, "-o", exe] + lk
        procs.append((exe, subprocess.Popen(cmd)))
    failed = [exe for exe, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"g++ {failed}")
    golden = os.path.join(ROOT, "tests", "golden")
    for d in DEMOS:
        out = subprocess.run([os.path.join(DROPIN, "ref_" + d)], check=True, capture_output=True,
                             text=True).stdout
        with open(os.path.join(golden, f"dropin_{d}.txt"), "w") as f:
            f.write(out)
    return [exe for exe, _ in procs]


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, prof="--prof" in sys.argv))
