for f in 0 4096 8192 12288; do CG_DEBUG_FLAGS=$f CG_BENCH_CHAIN=1 timeout 600 python bench.py --steps 504 --warmup 14 --no-cpu-baseline > gpurun_out/bench_f$f.json 2> gpurun_out/bench_f$f.err; tail -2 gpurun_out/bench_f$f.err
python -c "import json; d=json.load(open('gpurun_out/bench_f$f.json')); print($f, {k: d[k] for k in ('value','us_per_block','us_per_layer_staged_chain')})"; done
CG_DEBUG_FLAGS=4096 timeout 120 python tools/stamps_block.py | grep -E "previous|entry|prologue|pdl|task0 start|kernel end"
