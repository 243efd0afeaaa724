# fine stamps of one task switch (tools/micro/lib_fine.so: -DCG_FINE_STAMPS)
cp paper_2512_17970_b200/libcodegemm_b200.so /tmp/lib_cur.so
cp tools/micro/lib_fine.so paper_2512_17970_b200/libcodegemm_b200.so
FINE=1 timeout 300 python tools/stamps_block.py 2 2>&1 | grep -E "task[0-2] |fine"
cp /tmp/lib_cur.so paper_2512_17970_b200/libcodegemm_b200.so
