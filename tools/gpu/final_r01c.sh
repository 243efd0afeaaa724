# round-1 (third session) evidence: bench lines (8B default, 70B N=1, m2v8), ncu launch list and
# one full capture of the staged block kernel
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; tail -2 gpurun_out/bench_r01c.err
timeout 900 python bench.py --workload 70b --no-cpu-baseline > gpurun_out/bench_r01c_70b_n1.json 2> gpurun_out/bench_r01c_70b.err
timeout 900 python bench.py --config m2v8g128 --no-cpu-baseline > gpurun_out/bench_r01c_m2v8.json 2> gpurun_out/bench_r01c_m2v8.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -c 21 --csv --log-file gpurun_out/launches_r01c_block.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 4 -c 1 -o gpurun_out/prof_block_r01c -f python tools/stamps_block.py 2 > /dev/null 2>&1
timeout 300 python tools/stamps_block.py 2 > gpurun_out/stamps_block_r01c.txt 2>&1
ls -la gpurun_out/
