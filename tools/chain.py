"""Time dependent layer chains: separate launches (graph + PDL) vs one staged launch.

python tools/chain.py ROWS COLS [U]   -- a chain of same-shape layers
python tools/chain.py block [U]       -- the Llama-3-8B decoder block (4 stages)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
if sys.argv[1] == "block":
    u = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    shapes = [(4096, 4096, 0), (1024, 4096, 0), (1024, 4096, 0), (4096, 4096, 1),
              (14336, 4096, 2), (14336, 4096, 2), (4096, 14336, 3)]
    # reference suite multiplicity (bench.py): q,k,v,o 4096^2; gate, up; down
    shapes = [(4096, 4096, 0), (4096, 4096, 0), (4096, 4096, 0), (4096, 4096, 1),
              (14336, 4096, 2), (14336, 4096, 2), (4096, 14336, 3)]
else:
    rows, cols = int(sys.argv[1]), int(sys.argv[2])
    u = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    shapes = [(rows, cols, i) for i in range(7)]
per_step = sum(r * c * 0.265625 for r, c, _ in shapes)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
copies = max(2, int(np.ceil(3 * l2 / per_step)))
base = {}
for r, c, _ in shapes:
    if (r, c) not in base:
        base[(r, c)] = cg.random_layer(r, c, cfg, seed=r ^ c)
sets = [[cg.DeviceLayer(base[(r, c)], u=u) for r, c, _ in shapes] for _ in range(copies)]
xs = [torch.from_numpy(orc.bench_input_array(c, 1, i)).cuda() for i, (r, c, _) in enumerate(shapes)]
ys = [[torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, c, _ in shapes]
      for _ in range(copies)]
stages = [s for _, _, s in shapes]
print("u", sets[0][0].info["u"], "tasks", [L.info["n_tasks"] for L in sets[0]], "copies", copies)
s = torch.cuda.Stream()


def separate(k):
    grp = {}
    for i, st in enumerate(stages):
        grp.setdefault(st, []).append(i)
    for st in sorted(grp):
        ids = grp[st]
        cg.gemm_group([sets[k][i] for i in ids], [xs[i] for i in ids], [ys[k][i] for i in ids],
                      stream=s)


def staged(k):
    cg.gemm_stages(sets[k], xs, ys[k], stages, stream=s)


def time_it(fn):
    with torch.cuda.stream(s):
        for k in range(copies):
            fn(k)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for k in range(copies):
            fn(k)
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
    return e0.elapsed_time(e1) * 1e3 / (reps * copies)


ref = None
for name, fn in (("separate launches", separate), ("one staged launch", staged)):
    us = time_it(fn)
    out = [y.clone() for y in ys[0]]
    if ref is None:
        ref = out
    else:
        err = max(float((a - b).abs().max() / b.abs().max()) for a, b in zip(out, ref))
        print(f"  max normalised diff vs separate: {err:.2e}")
    print(f"{name:20s} {us:8.2f} us/step  {us / len(shapes):6.2f} us/layer  "
          f"{per_step / (us * 1e-6) / 1e9:8.1f} GB/s")
