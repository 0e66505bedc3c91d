# GPU perf round: correctness subset, benches per config, ncu launch list + full capture.
set -x
TAG=${TAG:-perf}
timeout 600 python -m pytest tests/test_gpu_adam.py tests/test_gpu_spmv.py -x -q 2>&1 | tail -3
for c in 1 2 3; do python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e > gpurun_out/${TAG}_c$c.json 2> gpurun_out/${TAG}_c$c.err; done
python bench.py --no-cpu > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_transpose" -s 6 -c 2 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/ncu2.log 2>&1
echo done
