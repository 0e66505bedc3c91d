#!/bin/bash
# A/B of the shared-memory window sweeps on the config-5 ensemble.
O=gpurun_out; mkdir -p $O
run() { env $1 $2 python bench.py --config ${3:-5} --steps 40 --warmup 5 --no-cpu --no-e2e --sustained-s 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$1 $2 groups', d['config']['restart_groups'], 'value %.0f apply_ms %.3f trans_ms %.3f' % (d['value'], k['apply']['ms_avg'], k['transpose']['ms_avg']))"; }
for g in 2 4; do
for v in 0 1 2 3 4; do run "CK_RESTART_GROUP=$g" "CK_WIN_TRANS=$v"; done
done | tee $O/ab_win.txt
run CK_X=1 CK_Y=1 4 | tee -a $O/ab_win.txt
run CK_T1_EARLY=1 CK_Y=1 4 | tee -a $O/ab_win.txt
run CK_X=1 CK_Y=1 4 | tee -a $O/ab_win.txt
run CK_T1_EARLY=1 CK_Y=1 4 | tee -a $O/ab_win.txt
