set -x
timeout 900 python -m pytest tests/test_xchg_gpu.py -x -q 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step']*1000, d['value'], d['roofline']['frac'])"
