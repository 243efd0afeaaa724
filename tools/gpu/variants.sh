set -x
timeout 300 python tools/variants.py 14336 4096 1
timeout 300 python tools/variants.py 14336 4096 2
timeout 300 python tools/variants.py 4096 4096 1
timeout 300 python tools/variants.py 28672 8192 1
timeout 120 python tools/stamps_group.py 14336 4096 1
