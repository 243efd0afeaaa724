cp paper_2512_17970_b200/libcodegemm_b200.so /tmp/lib_cur.so
cp tools/micro/lib_fine.so paper_2512_17970_b200/libcodegemm_b200.so
FINE=1 timeout 120 python tools/stamps_block.py 2 > gpurun_out/stamps_fine_r02d.txt 2>&1
cp /tmp/lib_cur.so paper_2512_17970_b200/libcodegemm_b200.so
grep -n "task1\|warp" gpurun_out/stamps_fine_r02d.txt | head -40
