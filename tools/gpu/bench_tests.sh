timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; tail -3 gpurun_out/bench_s.err
cat gpurun_out/bench_s.json
