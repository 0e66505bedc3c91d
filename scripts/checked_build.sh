#!/bin/bash
# Bounds-checked run of every device path (the stand-in for compute-sanitizer where the
# pool has it closed): rebuild libcondkit_b200.so with -DCK_CHECKED (device-side index
# assertions, ck_device.cuh), run the small cases and the parity tests that cover the
# window sweeps, the dense-block sweeps and the partition, then restore the product build.
# usage (GPU box): bash scripts/checked_build.sh OUT.txt
OUT=${1:-gpurun_out/checked.txt}
{
  echo "# checked build: -DCK_CHECKED"
  CK_NVCC_FLAGS=-DCK_CHECKED python -c "from paper_2409_11515_b200 import build; build.build(force=True)" 2>&1 | tail -2
  python scripts/sanitize_cases.py 12 2>&1 | tail -14
  timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_dist.py tests/test_gpu_inverse.py tests/test_gpu_adam.py tests/test_gpu_spmv.py -x -q 2>&1 | tail -4
  echo "# product build restored"
  python -c "from paper_2409_11515_b200 import build; build.build(force=True)" 2>&1 | tail -2
} > "$OUT" 2>&1
tail -12 "$OUT"
