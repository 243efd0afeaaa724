# stamps of the chained block, normal vs Psumbook build skipped (CG_DEBUG_FLAGS=256, timing only)
for f in 0 256; do echo "== flags $f"; CG_DEBUG_FLAGS=$f timeout 300 python tools/stamps_block.py 2 2>&1 | grep -E "task[0-7] (start|synced|x staged|table|gathered|task end)"; done
