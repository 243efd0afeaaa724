"""Where the end-to-end step's host time goes (diagnostics): wall clock per call of the
prepared 8B block launch with (a) launch + sync, (b) + H2D of the inputs, (c) + host
mirrors, and the same without the cooperative launch attribute (CG_DEBUG_FLAGS=4096)."""
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
layers = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 11 + i), u=4) for i, (_, r, c) in enumerate(spec)]
x0 = torch.from_numpy(orc.bench_input_array(4096, 1, 1)).cuda()
xbuf = torch.cat([x0.view(-1)] * 3)
xs_in = [xbuf[i * 4096:(i + 1) * 4096].view(4096, 1) for i in range(3)]
ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for _, r, c in spec]
xs = [xs_in[0], xs_in[1], xs_in[2], ys[0], ys[3], ys[3], ys[4]]
plan = cg.StagedLaunch(layers, xs, ys, list(bench.STEP_STAGES))
x_host = xbuf.cpu().pin_memory()
y_host = torch.empty(sum(y.numel() for y in ys)).pin_memory()
s = torch.cuda.current_stream()


def t(fn, n=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def launch_sync():
    plan()
    s.synchronize()


lib = plan._lib
print("launch only (no sync, us/call):", round(t(lambda: plan(), 300), 2))
print("launch + sync:", round(t(launch_sync), 2))
step_h2d = lambda: cg._lib.check(lib.cg_stages_run_host(plan.handle, x_host.data_ptr(), x_host.numel() * 2,  # noqa
                                                        xbuf.data_ptr(), None, None, 0, None))
print("H2D + launch + sync:", round(t(step_h2d), 2))
print("bind_host (H2D + launch + D2H + sync):",
      round(t(plan.bind_host(x_host, xbuf, torch.cat([y.view(-1) for y in ys]), y_host)), 2))
views, off = [], 0
for y in ys:
    views.append(y_host[off: off + y.numel()].view(y.shape))
    off += y.numel()
print("bind_host_mirrored (H2D + launch + sync):", round(t(plan.bind_host_mirrored(x_host, xbuf, views)), 2))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    plan()
e1.record()
torch.cuda.synchronize()
print("device us per launch (back to back):", round(e0.elapsed_time(e1) * 10, 2))
g = torch.cuda.CUDAGraph()
sg = torch.cuda.Stream()
with torch.cuda.stream(sg):
    plan(sg)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=sg):
    for _ in range(10):
        plan(sg)
with torch.cuda.stream(sg):
    for _ in range(3):
        g.replay()
    e0.record(sg)
    for _ in range(20):
        g.replay()
    e1.record(sg)
torch.cuda.synchronize()
print("device us per launch (graph of 10 launches, same weights):", round(e0.elapsed_time(e1) * 1e3 / 200, 2))
t0 = time.perf_counter()
for _ in range(100):
    plan._lib.cg_stages_launch(plan.handle, None)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host us per cg_stages_launch call (raw ctypes, default stream):", round((t1 - t0) * 1e4, 2),
      " total incl. drain:", round((t2 - t0) * 1e4, 2))
layers2 = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 911 + i), u=4) for i, (_, r, c) in enumerate(spec)]
ys2 = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for _, r, c in spec]
xs2 = [xs_in[0], xs_in[1], xs_in[2], ys2[0], ys2[3], ys2[3], ys2[4]]
plan2 = cg.StagedLaunch(layers2, xs2, ys2, list(bench.STEP_STAGES))
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(sg):
    plan2(sg)
torch.cuda.synchronize()
with torch.cuda.graph(g2, stream=sg):
    for _ in range(5):
        plan(sg)
        plan2(sg)
with torch.cuda.stream(sg):
    for _ in range(3):
        g2.replay()
    e0.record(sg)
    for _ in range(20):
        g2.replay()
    e1.record(sg)
torch.cuda.synchronize()
print("device us per launch (graph, two weight sets alternating):", round(e0.elapsed_time(e1) * 1e3 / 200, 2))
