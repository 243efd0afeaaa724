# main-kernel iteration: GPU tests of the fused path, the 8B/70B bench lines, block stamps
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_xchg_gpu.py -x -q > gpurun_out/r02_main_tests.txt 2>&1; tail -2 gpurun_out/r02_main_tests.txt
timeout 600 python bench.py --no-cpu-baseline --steps 500 --warmup 20 > gpurun_out/r02_main_bench.json 2> gpurun_out/r02_main_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r02_main_bench.json').read().strip().splitlines()[-1])
print('8b', d['us_per_block'], d['value'], d['roofline']['frac'], 'grouped', d['grouped_launches']['us_per_block'], 'sep', d['separate_launches']['us_per_block'], 'per-layer', d['us_per_layer'], 'e2e', d['e2e']['value'])"
timeout 300 python tools/stamps_block.py 2 > gpurun_out/r02_stamps_block.txt 2>&1; head -45 gpurun_out/r02_stamps_block.txt | tail -42
