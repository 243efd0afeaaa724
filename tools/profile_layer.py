"""Run a few fused GEMV launches of one layer shape (for ncu captures).

python tools/profile_layer.py --rows 14336 --cols 4096 --config m1v4g128 --iters 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

CONFIGS = {"m1v4g128": dict(v=4, m=1, b=8, g=128), "m2v8g128": dict(v=8, m=2, b=8, g=128),
           "m1v2b4g128": dict(v=2, m=1, b=4, g=128), "m2v4b4g128": dict(v=4, m=2, b=4, g=128),
           "m1v4b6g128": dict(v=4, m=1, b=6, g=128)}

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=14336)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--config", default="m1v4g128")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--u", type=int, default=0)
ap.add_argument("--rg", type=int, default=0)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--copies", type=int, default=4)
a = ap.parse_args()
c = CONFIGS[a.config]
qc = cg.QuantConfig(**c)
layers = [cg.DeviceLayer(cg.random_layer(a.rows, a.cols, qc, seed=s), u=a.u, rg_per_task=a.rg,
                         flags=a.flags) for s in range(a.copies)]
print(layers[0].info, flush=True)
x = torch.from_numpy(orc.bench_input_array(a.cols, a.batch, 0)).cuda()
y = torch.empty((a.rows, a.batch), dtype=torch.float32, device="cuda")
for i in range(a.iters):
    layers[i % len(layers)].gemm(x, y)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for i in range(200):
    layers[i % len(layers)].gemm(x, y)
ev[1].record()
torch.cuda.synchronize()
print(f"eager avg per call: {ev[0].elapsed_time(ev[1]) / 200 * 1e3:.2f} us", flush=True)
