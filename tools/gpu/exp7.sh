./tools/micro/cluster_occ
timeout 300 python tools/variants.py 14336 4096 1 full,skel-no-prefetch
CG_X_REGS=1 timeout 300 python tools/variants.py 14336 4096 1 full,skel-no-prefetch
