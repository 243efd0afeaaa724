"""Configuration sweeps on Llama-3-8B shapes.

python tools/sweep.py batch   -- m1v4g128, B in {1,4,8,16,32}
python tools/sweep.py hyper   -- (m, v, b) in {(1,4,8),(2,4,8),(1,8,8),(2,8,8),(3,8,8),(4,8,8),
                                  (1,2,4),(2,4,4),(1,4,6)} at g=128, B=1
Per shape: us per layer (graph of back-to-back staged chains, weights rotated > L2), HBM GB/s of
the algorithmic bytes, and a tolerance check against the C oracle on one call.
Prints one JSON line per (config, shape, batch).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import c_oracle  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

SHAPES = [("attn_proj", 4096, 4096), ("mlp_gate_up", 14336, 4096), ("mlp_down", 4096, 14336)]
L2 = torch.cuda.get_device_properties(0).L2_cache_size


def measure(cfg, rows, cols, n):
    qc = cg.QuantConfig(v=cfg["v"], m=cfg["m"], b=cfg["b"], g=cfg["g"])
    q0 = cg.random_layer(rows, cols, qc, seed=rows ^ cols)
    per = bench.layer_bytes(rows, cols, cfg, n, with_io=False)
    copies = max(2, int(np.ceil(3 * L2 / per)))
    layers = [cg.DeviceLayer(q0) for _ in range(copies)]
    info = layers[0].info
    if not info["fast_supported"]:
        return {"fast_supported": False}
    x16 = orc.bench_input_array(cols, n, 0)
    x = torch.from_numpy(x16).cuda()
    ys = [torch.empty((rows, n), dtype=torch.float32, device="cuda") for _ in range(copies)]
    # parity on one call
    y = layers[0].gemm(x).cpu().numpy()
    ref = c_oracle.codegemm([p.codes for p in q0.planes], [b.entries for b in q0.books],
                            q0.scales.scales, x16, cfg["v"], cfg["g"], threads=os.cpu_count())
    rel = float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-30))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for k in range(copies):
            layers[k].gemm(x, ys[k], stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for k in range(copies):
            layers[k].gemm(x, ys[k], stream=s)
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * copies)
    nbytes = bench.layer_bytes(rows, cols, cfg, n)
    return {"fast_supported": True, "u": info["u"], "us_per_layer": round(us, 3),
            "GBps": round(nbytes / (us * 1e-6) / 1e9, 1), "rel_l2_vs_oracle": rel,
            "bits_per_weight": round(8 * (bench.layer_bytes(rows, cols, cfg, n, False)) / (rows * cols), 4)}


mode = sys.argv[1] if len(sys.argv) > 1 else "batch"
if mode == "batch":
    cases = [(dict(v=4, m=1, b=8, g=128), n) for n in (1, 4, 8, 16, 32)]
else:
    cases = [(dict(v=v, m=m, b=b, g=128), 1) for (m, v, b) in
             ((1, 4, 8), (2, 4, 8), (1, 8, 8), (2, 8, 8), (3, 8, 8), (4, 8, 8), (1, 2, 4), (2, 4, 4),
              (1, 4, 6))]
for cfg, n in cases:
    for name, rows, cols in SHAPES:
        r = measure(cfg, rows, cols, n)
        r.update({"config": f"m{cfg['m']}v{cfg['v']}b{cfg['b']}g{cfg['g']}", "batch": n,
                  "shape": f"{name} {rows}x{cols}"})
        print(json.dumps(r), flush=True)
