"""Per-task phase timeline of the staged decoder-block launch (diagnostics).

python tools/stamps_block.py [8b|70b]   -- bench.py's N=1 step (u=2, q->o->gate/up->down)
Stamps of the last of a few launches; times in us from the first CTA start.
"""
import ctypes
import os
import sys

os.environ["CG_STAMPS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from paper_2512_17970_b200 import _lib  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "8b"
cfg = bench.CONFIGS["m1v4g128"]
spec = bench.block_spec(wl)
sets = [[cg.DeviceLayer(bench.make_layer(r, c, cfg, 7 * k + i), u=bench.TILING_U)
         for i, (_, r, c) in enumerate(spec)] for k in range(2)]
layers = sets[1]
xs0 = [torch.from_numpy(orc.bench_input_array(c, 1, i)).cuda() for i, (_, r, c) in enumerate(spec)]
ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for (_, r, c) in spec]
xs = [xs0[i] if src is None else ys[src] for i, src in enumerate(bench.STEP_XSRC)]
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    for k in range(2):
        cg.gemm_stages(sets[k], xs, ys, list(bench.STEP_STAGES), stream=s)
s.synchronize()
with torch.cuda.graph(g, stream=s):
    for k in range(2):
        cg.gemm_stages(sets[k], xs, ys, list(bench.STEP_STAGES), stream=s)
with torch.cuda.stream(s):
    for _ in range(3):
        g.replay()
torch.cuda.synchronize()
prev = np.zeros(torch.cuda.get_device_properties(0).multi_processor_count * 64, dtype=np.uint64)
sms = torch.cuda.get_device_properties(0).multi_processor_count
lib = _lib.load()
lib.cg_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
buf = np.zeros(sms * 64, dtype=np.uint64)
_lib.check(lib.cg_debug_stamps(layers[0].handle, buf.ctypes.data, sms * 64))
st = buf.reshape(sms, 64).astype(np.int64)
_lib.check(lib.cg_debug_stamps(sets[0][0].handle, prev.ctypes.data, sms * 64))
pv = prev.reshape(sms, 64).astype(np.int64)
t0 = st[st[:, 0] > 0, 0].min()
print(f"previous launch (same graph): last kernel end {(pv[:, 63].max() - t0) / 1e3:.2f} us")
print("tasks per layer", [L.info["n_tasks"] for L in layers])


def show(name, col):
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1000.0
        print(f"{name:22s} n={len(col):3d} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")


show("pdl_wait passed", st[:, 62])
names = [(0, "start"), (7, "synced"), (4, "inputs ok"), (5, "x staged"), (6, "table ready"), (1, "gathered"), (2, "zero ok/flush"),
         (3, "task end")]
for k in range(6):
    for slot, nm in names:
        show(f"task{k} {nm}", st[:, k * 8 + slot])
for b in range(3):
    for j, nm in enumerate(("entered", "drained", "arrived", "released")):
        show(f"barrier{b} {nm}", st[:, 48 + 4 * b + j])
show("kernel entry", st[:, 60])
show("prologue done", st[:, 61])
show("kernel end", st[:, 63])
