# L2 evict-first policy on streamed weights: A/B (CG_DEBUG_FLAGS=524288 = evict-normal)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
for e in "" "CG_DEBUG_FLAGS=524288" "" "CG_DEBUG_FLAGS=524288"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 1000 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e] chain8b', d['us_per_block'], d['roofline']['frac'], 'e2e', d['e2e']['value'])"
done
for e in "" "CG_DEBUG_FLAGS=524288"; do
  env $e timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 300 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e] chain70b', d['us_per_block'], d['roofline']['frac'])"
  env $e timeout 300 python tools/indep_block.py 8b 4 | sed "s/^/[$e] /"
done
timeout 120 python tools/stamps_block.py 2 > gpurun_out/stamps_evict.txt 2>&1; head -12 gpurun_out/stamps_evict.txt
