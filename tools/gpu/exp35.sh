for c in 1 2; do CG_BENCH_CHAIN=$c timeout 600 python bench.py --steps 504 --warmup 14 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -2 gpurun_out/bench_c$c.err
python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, {k: d[k] for k in ('value','us_per_block','gpu_launches','grouped_launches','separate_launches')})"; done
