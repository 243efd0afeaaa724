"""End-to-end step timing over rotating block copies (diagnostics): what bench.py's e2e does."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

cfg = bench.CONFIGS["m1v4g128"]
spec = bench.block_spec("8b")
x_host = torch.cat([torch.from_numpy(orc.bench_input_array(4096, 1, k)).view(-1) for k in range(3)]).pin_memory()
y_host = torch.empty(sum(r for _, r, c in spec)).pin_memory()
plans = []
for cp in range(7):
    layers = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 100 * cp + i), u=4) for i, (_, r, c) in enumerate(spec)]
    xbuf = torch.empty(3 * 4096, dtype=torch.float16, device="cuda")
    xs_in = [xbuf[i * 4096:(i + 1) * 4096].view(4096, 1) for i in range(3)]
    ybuf = torch.empty(sum(r for _, r, c in spec), device="cuda")
    ys, off = [], 0
    for _, r, c in spec:
        ys.append(ybuf[off:off + r].view(r, 1))
        off += r
    xs = [xs_in[0], xs_in[1], xs_in[2], ys[0], ys[3], ys[3], ys[4]]
    plan = cg.StagedLaunch(layers, xs, ys, list(bench.STEP_STAGES))
    views, off = [], 0
    for y in ys:
        views.append(y_host[off:off + y.numel()].view(y.shape))
        off += y.numel()
    plans.append((plan, plan.bind_host(x_host, xbuf, ybuf, y_host), plan.bind_host_mirrored(x_host, xbuf, views)))
for name, k in (("bind_host (H2D, launch, D2H, sync)", 1), ("mirrored (H2D, launch, sync)", 2)):
    for i in range(14):
        plans[i % 7][k]()
    t0 = time.perf_counter()
    n = 140
    for i in range(n):
        plans[i % 7][k]()
    dt = (time.perf_counter() - t0) / n
    print(f"{name}: {dt * 1e6:.1f} us per step")
