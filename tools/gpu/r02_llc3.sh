# LL chain per producer width: tests, then 8B/70B with CG_LL_CHAIN=0 / max 8 slices / max 64, one box
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for v in "CG_LL_CHAIN=0" "CG_LL_MAX_SLICES=8" "CG_LL_MAX_SLICES=64" "CG_LL_MAX_SLICES=16"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('8b $v', d['us_per_block'], d['roofline']['frac'])"
  env $v timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 1000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('70b $v', d['us_per_block'], d['roofline']['frac'])"
done
done
