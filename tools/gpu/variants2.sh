timeout 300 python tools/variants.py 14336 4096 1
timeout 300 python tools/variants.py 4096 4096 1
