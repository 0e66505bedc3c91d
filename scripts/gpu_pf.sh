timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pf_pytest.log 2>&1; tail -3 gpurun_out/pf_pytest.log
CK_TRACE=1 PYTHONPATH=. timeout 300 python scripts/trace_e2e.py 4 2>&1 | tail -12
timeout 600 python bench.py > gpurun_out/pf_b4.json 2> gpurun_out/pf_b4.err; python -c "
import json;d=json.load(open('gpurun_out/pf_b4.json'));print('value',d['value'],'e2e',d['e2e']['value'],'frac',d['roofline']['frac'],d['clocks'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
