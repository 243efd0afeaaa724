# ncu launch list of the bench step (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -c 30 --csv --log-file gpurun_out/launches.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
tail -2 gpurun_out/launches_bench.log
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches.csv')) if len(r)>10]
hdr=rows[0]; i=hdr.index('Metric Name'); v=hdr.index('Metric Value'); k=hdr.index('Kernel Name'); idx=hdr.index('ID')
from collections import defaultdict
d=defaultdict(dict)
for r in rows[1:]:
    d[r[idx]][r[i]]=r[v]; d[r[idx]]['k']=r[k][:60]
for key in list(d)[:30]:
    print(key, d[key]['k'], d[key].get('gpu__time_duration.sum'), d[key].get('dram__bytes_read.sum'))
PY
