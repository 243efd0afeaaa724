STAGED=1 U=2 timeout 100 python tools/stamps_group.py 14336 4096 3
STAGED=1 U=2 timeout 100 python tools/stamps_group.py 4096 4096 3
