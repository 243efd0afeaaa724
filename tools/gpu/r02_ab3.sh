# A/B of library builds on one box: 8B chain step (+ per-layer launches) and 70B (AB_VARIANTS = tools/micro/lib_<v>.so)
cp paper_2512_17970_b200/libcodegemm_b200.so /tmp/lib_cur.so
for rep in 1 2; do
for v in $AB_VARIANTS; do
  cp tools/micro/lib_$v.so paper_2512_17970_b200/libcodegemm_b200.so
  timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('8b $v', d['us_per_block'], d['roofline']['frac'], d['us_per_layer'], d['grouped_launches']['us_per_block'])"
  timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 500 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('70b $v', d['us_per_block'], d['roofline']['frac'])"
done
done
cp /tmp/lib_cur.so paper_2512_17970_b200/libcodegemm_b200.so
