mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_gemm -s 2 -c 1 -o gpurun_out/prof_batch_gateup_n4 -f python tools/profile_batch.py 14336 4096 4 > gpurun_out/prof_batch.log 2>&1; tail -3 gpurun_out/prof_batch.log
