# L2 prefetch of the next stage's task at task end: sweep CG_PF_NEXT on one box (8B and 70B blocks)
for rep in 1 2; do
for v in 0 2 4 8 16 64; do
  CG_PF_NEXT=$v timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('8b pf_next=$v', d['us_per_block'], d['roofline']['frac'])"
done
done
for v in 0 4 16 64; do
  CG_PF_NEXT=$v timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 1000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('70b pf_next=$v', d['us_per_block'], d['roofline']['frac'])"
done
