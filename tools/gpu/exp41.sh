for f in 0 2; do echo "flags $f"; CG_DEBUG_FLAGS=$f timeout 120 python tools/stamps_block.py | grep -E "previous|entry|pdl|prologue|task0 start|kernel end"; done
