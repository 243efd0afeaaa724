mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_grid_gpu.py -x -q > gpurun_out/r02_batch_tests.txt 2>&1; tail -3 gpurun_out/r02_batch_tests.txt
timeout 600 python tools/batch_sweep.py > gpurun_out/r02_batch_sweep.jsonl 2>&1; cat gpurun_out/r02_batch_sweep.jsonl | cut -c1-300
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_gemm -s 2 -c 1 -o gpurun_out/prof_batch_gateup_n4 -f python tools/profile_batch.py 14336 4096 4 > gpurun_out/prof_batch.log 2>&1; tail -1 gpurun_out/prof_batch.log
