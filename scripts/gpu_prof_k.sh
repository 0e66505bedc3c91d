set -x
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/k_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k_launches.csv $CMD > gpurun_out/k_ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_transpose" -s 6 -c 2 -o gpurun_out/k_prof_c4 $CMD > gpurun_out/k_ncu2.log 2>&1
echo rc=$?
timeout 600 python bench.py --config 5 --no-cpu > gpurun_out/k_b5.json 2> gpurun_out/k_b5.err; cat gpurun_out/k_b5.json
