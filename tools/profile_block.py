"""A few staged launches of bench.py's N=1 step (two chained 8B blocks, u = 4/m) for ncu.

python tools/profile_block.py [iters] [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "m1v4g128"]
u = 4 // cfg["m"]
spec = bench.block_spec("8b")
nl = len(spec)
sets = []
for k in range(2):  # two weight sets: consecutive launches stream different weights
    layers = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 100 * k + 7 * j + i), u=u)
              for j in range(2) for i, (_, r, c) in enumerate(spec)]
    ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for j in range(2)
          for (_, r, c) in spec]
    x0 = torch.from_numpy(orc.bench_input_array(spec[0][2], 1, k)).cuda()
    xs, st = [], []
    for j in range(2):
        for i, src in enumerate(bench.STEP_XSRC):
            xs.append(ys[j * nl + src] if src is not None else (x0 if j == 0 else ys[nl - 1]))
            st.append(4 * j + bench.STEP_STAGES[i])
    sets.append(cg.StagedLaunch(layers, xs, ys, st))
for it in range(iters):
    sets[it % 2]()
torch.cuda.synchronize()
print("ok")
