for i in 1 2 3; do
for m in early late; do
L=0; [ $m = late ] && L=1
echo "== $m $i"; CK_PF_PIN_LATE=$L CK_TRACE=1 PYTHONPATH=. timeout 300 python scripts/trace_e2e.py 4 2000 prefetch 2>&1 | tail -16
done; done
