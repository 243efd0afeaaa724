# LL consumer polling group A/B: default 16 partials per round; CG_DEBUG_FLAGS=1048576 = 8
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "staged or prepared or independent or chain" 2>&1 | tail -1
for rep in 1 2; do for e in "" "CG_DEBUG_FLAGS=1048576"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e] 8b', d['us_per_block'], d['roofline']['frac'], d['us_per_layer'])"
done; done
for e in "" "CG_DEBUG_FLAGS=1048576"; do
  env $e timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 500 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e] 70b', d['us_per_block'], d['roofline']['frac'])"
done
timeout 120 python tools/stamps_block.py 2 2>&1 | grep "task4 s\|task3 task end"
