for pf in 0 2 4 8; do
  CG_PF_DIST=$pf timeout 200 python tools/chain.py 28672 8192 4 | tail -1 | sed "s/^/pf=$pf 70B gate_up chain: /"
  CG_PF_DIST=$pf timeout 600 python bench.py --steps 504 --warmup 14 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf=$pf block8b', d['value'], d['us_per_block'])"
done
