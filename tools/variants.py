"""Per-launch time of the fused kernel under diagnostic phase switches (CG_DEBUG_FLAGS).

Graph replay over enough weight copies that the set exceeds L2; CUDA-event timing.
python tools/variants.py ROWS COLS [COUNT_IN_GROUP]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
group = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
base = cg.random_layer(rows, cols, cfg, seed=1)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
per = rows * cols * 0.265625 * group
copies = max(2, int(np.ceil(3 * l2 / per)))
layers = [[cg.DeviceLayer(base) for _ in range(group)] for _ in range(copies)]
x = torch.from_numpy(orc.bench_input_array(cols, 1, 0)).cuda()
ys = [[torch.empty((rows, 1), dtype=torch.float32, device="cuda") for _ in range(group)]
      for _ in range(copies)]
print(layers[0][0].info, "copies", copies, flush=True)
VARIANTS = [("full", 0), ("no-prefetch", 2), ("skip-build", 1 << 8), ("no-loads", 1 << 9),
            ("skip-gather", 1 << 10), ("skip-build+gather", (1 << 8) | (1 << 10)),
            ("skip-build,no-loads", (1 << 8) | (1 << 9)),
            ("skel-no-prefetch", (1 << 8) | (1 << 10) | 2),
            ("skel-determ", (1 << 8) | (1 << 10) | 16),
            ("empty", 1 << 11), ("empty-nocoop", (1 << 11) | (1 << 12)),
            ("full-nocoop", 1 << 12), ("empty-nopdl", (1 << 11) | (1 << 13)),
            ("empty-nopdl-nocoop", (1 << 11) | (1 << 12) | (1 << 13)), ("full-nopdl", 1 << 13)]
if len(sys.argv) > 4:
    VARIANTS = [v for v in VARIANTS if v[0] in sys.argv[4].split(",")]
s = torch.cuda.Stream()
for name, fl in VARIANTS:
    os.environ["CG_DEBUG_FLAGS"] = str(fl)
    with torch.cuda.stream(s):
        for c in range(copies):
            cg.gemm_group(layers[c], [x] * group, ys[c], stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for c in range(copies):
            cg.gemm_group(layers[c], [x] * group, ys[c], stream=s)
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * copies)
    gbs = per / (us * 1e-6) / 1e9
    print(f"{name:22s} {us:8.2f} us/launch  {gbs:8.1f} GB/s", flush=True)
os.environ["CG_DEBUG_FLAGS"] = "0"
