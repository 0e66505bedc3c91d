#!/bin/bash
# One GPU evidence pass: tests, bench lines, ncu launch list + full capture, sanitizer.
# usage: gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh TAG [notest]'
TAG=${1:-r02x}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/${TAG}_gpu.txt
if [ "$2" != "notest" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.txt 2>&1
  tail -3 $O/${TAG}_pytest.txt
fi
python bench.py --steps 300 --warmup 10 > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err; tail -c 1500 $O/${TAG}_bench_c4.json
python bench.py --config 5 --steps 100 --warmup 5 --no-cpu > $O/${TAG}_bench_c5.json 2> $O/${TAG}_bench_c5.err; tail -c 1200 $O/${TAG}_bench_c5.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_reference_arm_c4.json 2> $O/${TAG}_ref.err; tail -c 600 $O/${TAG}_reference_arm_c4.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches_c4.csv \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_apply|k_transpose' -s 10 -c 2 -f -o $O/${TAG}_full_c4 \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_ncu_full_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_apply|k_transpose' -s 10 -c 2 -f -o $O/${TAG}_full_c5 \
  python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_ncu_full_c5.log 2>&1
ls -la $O
CK_TRACE=1 python scripts/trace_e2e.py 4 > $O/${TAG}_trace_e2e_c4.txt 2>&1
python bench.py --partition --steps 100 --warmup 5 --no-cpu --no-e2e > $O/${TAG}_bench_partition_ws1.json 2> $O/${TAG}_part.err; tail -c 400 $O/${TAG}_bench_partition_ws1.json
python __graft_entry__.py > $O/${TAG}_smoke.txt 2>&1; tail -1 $O/${TAG}_smoke.txt
