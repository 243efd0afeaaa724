timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/stamps_block.py | grep -E "tasks per|task[0-9] (start|table|gathered|task end)|released|kernel end"
timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; tail -3 gpurun_out/bench_s.err
python -c "import json; d=json.load(open('gpurun_out/bench_s.json')); print({k: d[k] for k in ('value','us_per_block','us_per_layer','us_per_layer_staged_chain','grouped_launches','separate_launches','e2e')})"
