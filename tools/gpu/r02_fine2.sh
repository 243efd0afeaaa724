# fine stamps (lib_fine) and the 8B bench with the current library
bash tools/gpu/r02_fine.sh | grep -E "task0 task end|task1"
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('8b', d['us_per_block'], d['roofline']['frac'])"
CG_LL_CHAIN=0 timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('8b nollc', d['us_per_block'], d['roofline']['frac'])"
done
