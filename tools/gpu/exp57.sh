timeout 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CG_ROW_DEPS=1 timeout 800 python -m pytest tests -m gpu -x -q -k staged 2>&1 | tail -2
timeout 600 python bench.py --steps 504 --warmup 14 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['us_per_block'])"
