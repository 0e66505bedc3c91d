set -x
for i in 1 2; do
CK_LIB=$PWD/ab_novec.so timeout 300 python bench.py --config 5 --no-cpu --no-e2e > gpurun_out/ab_novec_$i.json 2>&1
timeout 300 python bench.py --config 5 --no-cpu --no-e2e > gpurun_out/ab_vec_$i.json 2>&1
done
for f in gpurun_out/ab_*.json; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);k=d['kernels'];print('$f',round(d['value']),k['apply']['ms_avg'],k['transpose']['ms_avg'])"; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; tail -3 gpurun_out/ab_pytest.log
