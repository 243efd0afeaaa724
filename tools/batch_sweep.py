"""Batch sweep (BASELINE config 4): 8B block layers at n = 1/2/4/8/16/32, device time.

python tools/batch_sweep.py [config] [--lookups]
One JSON line per batch size: per-shape us (graphs of back-to-back launches
over rotating weight copies larger than L2), the block sum with multiplicities,
GB/s of algorithmic bytes, and which kernel ran (n = 1: fused Psumbook lookups;
n >= 2: the K4 batch kernel, or -- with --lookups -- one Psumbook per column).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from paper_2512_17970_b200 import _lib  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

cfg_name = next((a for a in sys.argv[1:] if not a.startswith("--")), "m1v4g128")
lookups = "--lookups" in sys.argv
cfg = bench.CONFIGS[cfg_name]
shapes = [(name, r, c, mult) for (name, r, c, mult) in bench.SUITES["8b"]]
flags = _lib.CG_OPT_NO_BATCH if lookups else 0
COPIES = 6
layers = {}
for name, r, c, _ in shapes:
    layers[name] = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 17 * k + r), flags=flags)
                    for k in range(COPIES)]
s = torch.cuda.Stream()
for n in (1, 2, 4, 8, 16, 32):
    per = {}
    for name, r, c, mult in shapes:
        xs = [torch.from_numpy(orc.bench_input_array(c, n, k)).cuda() for k in range(COPIES)]
        ys = [torch.empty((r, n), dtype=torch.float32, device="cuda") for _ in range(COPIES)]
        dls = layers[name]
        with torch.cuda.stream(s):
            for k in range(COPIES):
                dls[k].gemm(xs[k], ys[k])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for k in range(COPIES):
                dls[k].gemm(xs[k], ys[k])
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        per[name] = e0.elapsed_time(e1) * 1e3 / (reps * COPIES)
    block_us = sum(per[nm] * mult for nm, r, c, mult in shapes)
    block_bytes = sum(bench.layer_bytes(r, c, cfg, n) * mult for nm, r, c, mult in shapes)
    kernel = ("fused Psumbook lookups" if n == 1 or lookups else "K4 batch (mma.sync dequant)")
    print(json.dumps({"config": cfg_name, "batch": n, "kernel": kernel,
                      "us_per_layer": {f"{nm} {r}x{c}": round(per[nm], 2) for nm, r, c, _ in shapes},
                      "block_us_sum": round(block_us, 2),
                      "block_GBps": round(block_bytes / (block_us * 1e-6) / 1e9, 1),
                      "frac_of_measured_hbm": round(block_bytes / (block_us * 1e-6) / 1e9 / 6538.3, 4)}),
          flush=True)
