# final bench lines of the round (HEAD library = r02e kernels; bench.py with the pre-start spin)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02f2_tests.txt 2>&1; tail -1 gpurun_out/r02f2_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bench_r02g_k20.json 2>/dev/null
timeout 900 python bench.py --workload 70b --no-cpu-baseline --no-extras > gpurun_out/bench_r02g_70b_n1.json 2> /dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02g.json 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/bench_r02g.json", "gpurun_out/bench_r02g_k20.json", "gpurun_out/bench_r02g_70b_n1.json", "gpurun_out/bench_ref_r02g.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("us_per_block"), (d.get("roofline") or {}).get("frac"), d.get("e2e", {}).get("value"), d.get("gpu_launches"))
    except Exception as e:
        print(f, "ERR", e)
PY
