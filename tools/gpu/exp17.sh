STAGED=1 U=2 timeout 100 python tools/stamps_group.py 14336 4096 2 | grep -E "task1|released|arrived"
timeout 200 python tools/chain.py block 2
timeout 200 python tools/chain.py 14336 4096 2
timeout 200 python tools/chain.py 14336 4096 4
