set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --config 3 --steps 200 --warmup 10 --no-cpu > gpurun_out/b3.json 2> gpurun_out/b3.err
python bench.py > gpurun_out/b4.json 2> gpurun_out/b4.err
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
$CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_transpose" -s 6 -c 2 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu2.log 2>&1
echo rc=$?
