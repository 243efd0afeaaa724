cp paper_2512_17970_b200/libcodegemm_b200.so /tmp/lib_cur.so
for v in old new2; do
  cp tools/micro/lib_$v.so paper_2512_17970_b200/libcodegemm_b200.so
  echo "== $v"; timeout 120 python tools/stamps_block.py 2 2>&1 | head -64 | awk 'NR<=12 || /task1|task2|kernel end/'
  timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 2000 > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('8b $v', d['us_per_block'], d['roofline']['frac'], d['us_per_layer'])"
done
cp /tmp/lib_cur.so paper_2512_17970_b200/libcodegemm_b200.so
