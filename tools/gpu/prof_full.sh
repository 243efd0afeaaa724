# GPU-box script: one ncu --set full capture of the fused kernel on a layer shape
# usage: bash tools/gpu/prof_full.sh NAME ROWS COLS [extra profile_layer args]
name=$1; rows=$2; cols=$3; shift 3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 8 -c 1 \
    -o gpurun_out/$name -f python tools/profile_layer.py --rows $rows --cols $cols --iters 10 "$@" \
    > gpurun_out/$name.log 2>&1
tail -3 gpurun_out/$name.log
