cp paper_2512_17970_b200/libcodegemm_b200.so /tmp/lib_cur.so
cp tools/micro/lib_fine.so paper_2512_17970_b200/libcodegemm_b200.so
for f in 0 256; do echo "== flags $f"; CG_DEBUG_FLAGS=$f FINE=1 timeout 300 python tools/stamps_block.py 2 2>&1 | grep -E "task1 |fine"; done
cp /tmp/lib_cur.so paper_2512_17970_b200/libcodegemm_b200.so
