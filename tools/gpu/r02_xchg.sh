mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_xchg_gpu.py -x -q 2>&1 | tail -3
timeout 600 python tools/xchg_bench.py 8b > gpurun_out/xchg_bench_r02_8b.json 2>&1; tail -c 1500 gpurun_out/xchg_bench_r02_8b.json
CG_XC_LL=0 timeout 600 python tools/xchg_bench.py 8b > gpurun_out/xchg_bench_r02_8b_fenced.json 2>&1; tail -c 600 gpurun_out/xchg_bench_r02_8b_fenced.json
