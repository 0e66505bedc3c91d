#!/bin/bash
# A/B of the window sweeps on the config-5 ensemble: global gathers vs the shared-memory
# window, restart groups of 2 and 4 columns, and the library's default choice.
O=gpurun_out; mkdir -p $O
run() { env $1 $2 python bench.py --config ${3:-5} --steps 40 --warmup 5 --no-cpu --no-e2e --sustained-s 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('$1 $2 groups', d['config']['restart_groups'], 'value %.0f apply_ms %.3f trans_ms %.3f' % (d['value'], k['apply']['ms_avg'], k['transpose']['ms_avg']))"; }
for g in 2 4; do
for v in CK_NO_WINDOW=1 CK_WINDOW=default; do run "CK_RESTART_GROUP=$g" "$v"; done
done | tee $O/ab_win.txt
run CK_DEFAULT=1 CK_WINDOW=default | tee -a $O/ab_win.txt
