# GPU-box script: gpu tests + stamps of the fused kernel + short per-shape timing
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 120 python tools/stamps_group.py 14336 4096 2
timeout 120 python tools/stamps_group.py 4096 4096 3
timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --detail > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -3 gpurun_out/bench_q.err
cat gpurun_out/bench_q.json
