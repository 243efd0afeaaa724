mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_tests_sub.txt 2>&1; tail -2 gpurun_out/r02_tests_sub.txt
timeout 900 python tools/sweep.py hyper > gpurun_out/sweep_hyper_r02.jsonl 2>&1; cut -c1-220 gpurun_out/sweep_hyper_r02.jsonl
for c in m1v2b4g128 m2v4b4g128 m1v4b6g128 m1v4g128; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:group_gemv -s 3 -c 1 --csv python tools/profile_layer.py --rows 14336 --cols 4096 --config $c --iters 5 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' -v c=$c '{print c, $(NF-2), $NF}'
done
