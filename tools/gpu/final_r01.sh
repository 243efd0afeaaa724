# round-1 evidence: default bench line, reference arm, ncu launch list + full capture of the staged block kernel
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -2 gpurun_out/bench_r01.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01.json 2> gpurun_out/bench_ref_r01.err; tail -1 gpurun_out/bench_ref_r01.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -c 21 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 4 -c 1 -o gpurun_out/prof_block_r01 -f python tools/stamps_block.py > /dev/null 2>&1
ls -la gpurun_out/
