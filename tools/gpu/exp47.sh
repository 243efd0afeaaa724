for c in 1 2; do CG_BENCH_CHAIN=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:group_gemv -c 8 --csv --log-file gpurun_out/l$c.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/l$c.csv')) if len(r)>10]
h=rows[0]; v=h.index('Metric Value')
print($c, [r[v] for r in rows[1:]])
PY
done
