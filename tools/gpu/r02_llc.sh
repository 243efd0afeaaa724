# LL chain: GPU tests, then an A/B of CG_LL_CHAIN=0/1 on one box (bench.py's 8B step)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for rep in 1 2; do
for v in 0 1; do
  CG_LL_CHAIN=$v timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('llc=$v', d['us_per_block'], d['roofline']['frac'], d.get('e2e',{}).get('value'))"
done
done
