"""Experiment: the 8B/70B block's 7 layers as INDEPENDENT layers (the reference
bench protocol, /root/reference/pkg/src/codegemm/bench.py:192-214: every layer
timed on its own input) in one persistent launch -- one stage, no grid barriers
-- against the staged decode chain.  Prints one JSON line per variant.

usage: python tools/indep_block.py [8b|70b] [u]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402  (input generator only)

wl = sys.argv[1] if len(sys.argv) > 1 else "8b"
u = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = bench.CONFIGS["m1v4g128"]
spec = bench.block_spec(wl)
dev = torch.device("cuda", 0)
wbytes = sum(bench.layer_bytes(r, c, cfg, 1, with_io=False) for _, r, c in spec)
abytes = sum(bench.layer_bytes(r, c, cfg, 1) for _, r, c in spec)
copies = max(2, -(-3 * bench.L2_BYTES // wbytes))
peak = 6538.3
blocks = []
for cp in range(copies):
    lay = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 91_000 + 100 * cp + i), u=u)
           for i, (_, r, c) in enumerate(spec)]
    xs = [torch.from_numpy(orc.bench_input_array(c, 1, 10 * cp + i)).to(dev)
          for i, (_, r, c) in enumerate(spec)]
    ys = [torch.empty((r, 1), dtype=torch.float32, device=dev) for _, r, c in spec]
    blocks.append((lay, xs, ys))

stream = torch.cuda.Stream(dev)


def capture(fn):
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def time_graph(g, reps):
    with torch.cuda.stream(stream):
        for _ in range(5):
            g.replay()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / reps * 1e3  # us per replay


def report(name, us_per_block, extra=None):
    d = {"variant": name, "workload": wl, "u": u, "us_per_block": round(us_per_block, 3),
         "GB/s": round(abytes / (us_per_block * 1e-6) / 1e9, 1),
         "frac": round(abytes / (us_per_block * 1e-6) / 1e9 / peak, 4)}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


# (a) one launch per block, all 7 layers independent (one stage)
plans = [cg.StagedLaunch(lay, xs, ys, [0] * len(lay)) for lay, xs, ys in blocks]
g = capture(lambda: [p() for p in plans])
report("indep_one_stage", time_graph(g, 200) / copies)
del g, plans
# (b) two blocks per launch, independent (14 layers, one stage)
if len(spec) * 2 <= 16:
    plans = [cg.StagedLaunch(blocks[j][0] + blocks[j + 1][0], blocks[j][1] + blocks[j + 1][1],
                             blocks[j][2] + blocks[j + 1][2], [0] * (2 * len(spec)))
             for j in range(0, copies - 1, 2)]
    g = capture(lambda: [p() for p in plans])
    report("indep_two_blocks_one_stage", time_graph(g, 200) / (2 * len(plans)))
    del g, plans
# (c) the decode chain, one launch per block
stages = list(bench.STEP_STAGES)
plans = []
for lay, xs, ys in blocks:
    xx = [xs[i] if src is None else ys[src] for i, src in enumerate(bench.STEP_XSRC)]
    plans.append(cg.StagedLaunch(lay, xx, ys, stages))
g = capture(lambda: [p() for p in plans])
report("chain_one_block", time_graph(g, 200) / copies)
