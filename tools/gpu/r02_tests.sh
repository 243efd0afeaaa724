mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02_tests.txt 2>&1; tail -25 gpurun_out/r02_tests.txt
