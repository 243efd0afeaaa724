# independent-layer launches (reference protocol) vs the decode chain
mkdir -p gpurun_out
for a in "8b 4" "8b 2" "70b 4" "70b 2"; do timeout 300 python tools/indep_block.py $a; done > gpurun_out/indep.jsonl 2> gpurun_out/indep.err
CG_DEBUG_FLAGS=256 timeout 300 python tools/indep_block.py 8b 4 > gpurun_out/indep_nobuild.jsonl 2>&1
cat gpurun_out/indep.jsonl gpurun_out/indep_nobuild.jsonl; tail -3 gpurun_out/indep.err
