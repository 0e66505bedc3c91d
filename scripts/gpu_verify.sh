set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; tail -3 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_b4.json 2> gpurun_out/v_b4.err; cat gpurun_out/v_b4.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err; cat gpurun_out/v_ref.json
echo done
