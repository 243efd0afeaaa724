"""Staged launches of a chain of same-shape layers (for ncu captures).

python tools/profile_chain.py ROWS COLS COUNT U [ITERS]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

rows, cols, count, u = (int(a) for a in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 10
cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
sets = [[cg.DeviceLayer(cg.random_layer(rows, cols, cfg, seed=10 * k + i), u=u) for i in range(count)]
        for k in range(4)]
x = torch.from_numpy(orc.bench_input_array(cols, 1, 0)).cuda()
ys = [torch.empty((rows, 1), dtype=torch.float32, device="cuda") for _ in range(count)]
xs = [x] * count
for it in range(iters):
    cg.gemm_stages(sets[it % 4], xs, ys, list(range(count)))
torch.cuda.synchronize()
print("done", sets[0][0].info)
