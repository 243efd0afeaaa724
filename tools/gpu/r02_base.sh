# round 2: baseline of the round-1 state on a fresh box (tests + bench)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_base_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_base_tests.txt 2>&1; tail -3 gpurun_out/r02_base_tests.txt
timeout 600 python bench.py > gpurun_out/r02_base_bench.json 2> gpurun_out/r02_base_bench.err; tail -c 600 gpurun_out/r02_base_bench.json
