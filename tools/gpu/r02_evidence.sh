# round-2 evidence: bench lines, ncu launch list + full captures, sweeps, exchange bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r02e_smi.txt
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -2 gpurun_out/bench_r02.err
timeout 900 python bench.py --workload 70b --no-cpu-baseline --no-extras > gpurun_out/bench_r02_70b_n1.json 2> gpurun_out/bench_r02_70b.err
timeout 900 python bench.py --config m2v8g128 --no-cpu-baseline --no-extras > gpurun_out/bench_r02_m2v8.json 2> gpurun_out/bench_r02_m2v8.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -c 21 --csv --log-file gpurun_out/launches_r02_block.csv python bench.py --steps 14 --warmup 7 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 2 -c 1 -o gpurun_out/prof_block_r02 -f python tools/profile_block.py 4 > /dev/null 2>&1
CG_DEBUG_FLAGS=256 timeout 900 ncu --set full --clock-control none -k regex:group_gemv -s 3 -c 1 -o gpurun_out/prof_gather_only_r02 -f python tools/profile_layer.py --rows 28672 --cols 8192 --iters 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:group_gemv -s 3 -c 1 -o gpurun_out/prof_70b_gateup_r02 -f python tools/profile_layer.py --rows 28672 --cols 8192 --iters 5 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_gemm -s 2 -c 1 -o gpurun_out/prof_batch_n8_r02 -f python tools/profile_batch.py 14336 4096 8 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:batch_gemm -s 2 -c 1 -o gpurun_out/prof_batch_n32_r02 -f python tools/profile_batch.py 14336 4096 32 > /dev/null 2>&1
timeout 900 python tools/batch_sweep.py m1v4g128 > gpurun_out/sweep_batch_r02.jsonl 2>&1
timeout 900 python tools/batch_sweep.py m2v8g128 >> gpurun_out/sweep_batch_r02.jsonl 2>&1
timeout 900 python tools/xchg_bench.py 70b > gpurun_out/xchg_bench_r02_70b.json 2>&1
CG_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_r02_onegpu_2ranks.json 2> gpurun_out/bench_r02_onegpu_2ranks.err; tail -c 300 gpurun_out/bench_r02_onegpu_2ranks.json

# ncu reports -> CSV (raw metrics; source lines for the block and batch captures), reports removed
for r in prof_block_r02 prof_gather_only_r02 prof_70b_gateup_r02 prof_batch_n8_r02 prof_batch_n32_r02; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
for r in prof_block_r02 prof_batch_n8_r02; do
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${r}_source.csv 2>/dev/null
done
python tools/ncu_lines.py gpurun_out/prof_block_r02_source.csv 0.01 > gpurun_out/ncu_lines_r02_block.txt 2>&1
python tools/ncu_lines.py gpurun_out/prof_batch_n8_r02_source.csv 0.01 > gpurun_out/ncu_lines_r02_batch_n8.txt 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/*_source.csv
du -sh gpurun_out
