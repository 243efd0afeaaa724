timeout 100 python tools/stamps_group.py 14336 4096 1
timeout 100 python tools/stamps_group.py 14336 4096 1 1282
timeout 100 python tools/stamps_group.py 4096 4096 1
