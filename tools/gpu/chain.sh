timeout 200 python tools/chain.py block 2
timeout 200 python tools/chain.py block 4
timeout 200 python tools/chain.py 14336 4096 2
timeout 200 python tools/chain.py 14336 4096 4
timeout 200 python tools/chain.py 4096 4096 2
timeout 200 python tools/chain.py 28672 8192 4
