# evidence of the final library (LL limit 32): tests, bench lines, reference arm, ncu launch list + full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_tests.txt 2>&1; tail -1 gpurun_out/r02h_tests.txt
timeout 900 python bench.py > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err; tail -2 gpurun_out/bench_r02h.err
timeout 900 python bench.py --workload 70b --no-cpu-baseline --no-extras > gpurun_out/bench_r02h_70b_n1.json 2> gpurun_out/bench_r02h_70b.err
timeout 900 python bench.py --config m2v8g128 --no-cpu-baseline --no-extras > gpurun_out/bench_r02h_m2v8.json 2> gpurun_out/bench_r02h_m2v8.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02h.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -c 21 --csv --log-file gpurun_out/launches_r02h_block.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 2 -c 1 -o gpurun_out/prof_block_r02h -f python tools/profile_block.py 4 > /dev/null 2>&1
ncu -i gpurun_out/prof_block_r02h.ncu-rep --page raw --csv > gpurun_out/prof_block_r02h_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_block_r02h.ncu-rep --page details --csv > gpurun_out/prof_block_r02h_details.csv 2>/dev/null
ncu -i gpurun_out/prof_block_r02h.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/prof_block_r02h_source.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/prof_block_r02h_source.csv 0.01 > gpurun_out/ncu_lines_r02h_block.txt 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/*_source.csv
timeout 120 python tools/stamps_block.py 2 > gpurun_out/stamps_block_r02h.txt 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/bench_r02h.json", "gpurun_out/bench_r02h_70b_n1.json", "gpurun_out/bench_r02h_m2v8.json", "gpurun_out/bench_ref_r02h.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("us_per_block"), (d.get("roofline") or {}).get("frac"), d.get("e2e", {}).get("value"), d.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_r02h_k20.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_r02h_k20.json').read().strip().splitlines()[-1]); print('k20', d['value'], d['ms_per_step'], d['roofline']['frac'])"
