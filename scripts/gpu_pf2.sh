for i in 1 2 3; do
for m in none prefetch; do
echo "== $m $i"; CK_TRACE=1 PYTHONPATH=. timeout 300 python scripts/trace_e2e.py 4 2000 $m 2>&1 | grep -v SELL | tail -9
done; done
