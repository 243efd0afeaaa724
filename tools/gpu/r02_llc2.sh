# LL chain: stamps of the chained block (on/off), 70B A/B
for v in 1 0; do
  echo "== CG_LL_CHAIN=$v"; CG_LL_CHAIN=$v timeout 300 python tools/stamps_block.py 2 2>&1 | grep -v barrier | head -75
done
for rep in 1 2; do
for v in 0 1; do
  CG_LL_CHAIN=$v timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 1000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('70b llc=$v', d['us_per_block'], d['roofline']['frac'])"
done
done
