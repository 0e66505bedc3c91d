for i in 1 2; do
for v in base w1 w2 w3 w4; do
  if [ $v = base ]; then L=$PWD/paper_2409_11515_b200/libcondkit_b200.so; else L=$PWD/ab_$v.so; fi
  CK_LIB=$L timeout 300 python bench.py --config 5 --no-cpu --no-e2e > gpurun_out/abt_${v}_$i.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/abt_${v}_$i.json').read().strip().splitlines()[-1]);k=d['kernels'];print('$v $i',round(d['value']),k['apply']['ms_avg'],k['transpose']['ms_avg'])"
done; done
