# round-2 final evidence (HEAD): tests, bench lines, reference arm, ncu launch list + full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r02c_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_tests.txt 2>&1; tail -2 gpurun_out/r02c_tests.txt
timeout 900 python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; tail -2 gpurun_out/bench_r02c.err
timeout 900 python bench.py --workload 70b --no-cpu-baseline --no-extras > gpurun_out/bench_r02c_70b_n1.json 2> gpurun_out/bench_r02c_70b.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02c.json 2>&1
timeout 300 python tools/indep_block.py 70b 4 > gpurun_out/indep_r02c_70b.jsonl 2>&1
timeout 300 python tools/indep_block.py 8b 4 > gpurun_out/indep_r02c_8b.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -c 21 --csv --log-file gpurun_out/launches_r02c_block.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 2 -c 1 -o gpurun_out/prof_block_r02c -f python tools/profile_block.py 4 > /dev/null 2>&1
for r in prof_block_r02c; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${r}_source.csv 2>/dev/null
done
python tools/ncu_lines.py gpurun_out/prof_block_r02c_source.csv 0.01 > gpurun_out/ncu_lines_r02c_block.txt 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/*_source.csv
python - <<'PY'
import json
for f in ["gpurun_out/bench_r02c.json", "gpurun_out/bench_r02c_70b_n1.json", "gpurun_out/bench_ref_r02c.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), d.get("e2e", {}).get("value"), d.get("independent_layers"), d.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
cat gpurun_out/indep_r02c_70b.jsonl gpurun_out/indep_r02c_8b.jsonl
du -sh gpurun_out
