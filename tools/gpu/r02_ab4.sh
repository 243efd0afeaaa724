timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
AB_VARIANTS="old t" bash tools/gpu/r02_ab3.sh
for v in old t; do cp tools/micro/lib_$v.so paper_2512_17970_b200/libcodegemm_b200.so; timeout 300 python tools/indep_block.py 70b 4 | sed "s/^/$v /"; done
cp tools/micro/lib_t.so paper_2512_17970_b200/libcodegemm_b200.so
