# GPU-box script: tests, bench, per-phase stamps of the fused kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --detail > gpurun_out/bench_cur.json 2> gpurun_out/bench_cur.err; tail -3 gpurun_out/bench_cur.err
cat gpurun_out/bench_cur.json
timeout 120 python tools/stamps_group.py 14336 4096 2
timeout 120 python tools/stamps.py 14336 4096
timeout 120 python tools/stamps.py 4096 4096
