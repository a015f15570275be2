# small batches: one walk per lane (no budget) vs every query parked at once into the CTA pass
for v in "X=0" "FKD_BUDGET=1" "X=0" "FKD_BUDGET=1"; do
  echo "== $v"; env $v python tools/latency.py 2>&1 | grep -v '"m": 100000'
done
