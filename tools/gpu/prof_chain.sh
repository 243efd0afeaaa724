# usage: bash tools/gpu/prof_chain.sh NAME ROWS COLS COUNT U
name=$1; shift
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 6 -c 1 \
    -o gpurun_out/$name -f python tools/profile_chain.py "$@" > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log
