mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "staged or prepared or independent" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 1000 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chain8b', d['us_per_block'], d['roofline']['frac'], d['e2e']['value'])"
timeout 120 python tools/stamps_block.py 2 > gpurun_out/stamps_prol.txt 2>&1; head -12 gpurun_out/stamps_prol.txt
