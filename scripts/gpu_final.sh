timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; tail -1 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/f_b4.json 2> gpurun_out/f_b4.err; python -c "
import json;d=json.load(open('gpurun_out/f_b4.json'));print('value',d['value'],'e2e',d['e2e']['value'],'frac',d['roofline']['frac'],d['clocks'])"
