# LL chain producer slice limit A/B (CG_LL_MAX_SLICES; default 8)
for e in "" "CG_LL_MAX_SLICES=16" "CG_LL_MAX_SLICES=32" "CG_LL_MAX_SLICES=64" ""; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e] 8b', d['us_per_block'], d['roofline']['frac'])"
  env $e timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 500 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e] 70b', d['us_per_block'], d['roofline']['frac'])"
done
