mkdir -p gpurun_out
INDEP=1 timeout 120 python tools/stamps_block.py 1 > gpurun_out/stamps_indep1.txt 2>&1
INDEP=1 timeout 120 python tools/stamps_block.py 2 > gpurun_out/stamps_indep2.txt 2>&1
head -60 gpurun_out/stamps_indep1.txt; echo ====; head -60 gpurun_out/stamps_indep2.txt
