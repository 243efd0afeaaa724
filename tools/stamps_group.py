"""Per-task phase timeline of a grouped launch (diagnostics; CG_STAMPS=1).

python tools/stamps_group.py ROWS COLS COUNT [CG_DEBUG_FLAGS]
Runs a few launches back to back (graph of 4 launches, PDL) and prints the
stamps of the last one, relative to the earliest CTA start of that launch.
"""
import ctypes
import os
import sys

os.environ["CG_STAMPS"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17970_b200 as cg  # noqa: E402
from paper_2512_17970_b200 import _lib  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

rows, cols, count = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
if len(sys.argv) > 4:
    os.environ["CG_DEBUG_FLAGS"] = sys.argv[4]
staged = os.environ.get("STAGED", "0") == "1"  # count layers as a dependent chain
u = int(os.environ.get("U", "0"))
cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
sets = [[cg.DeviceLayer(cg.random_layer(rows, cols, cfg, seed=i), u=u) for i in range(count)]
        for _ in range(2)]
ys = [torch.empty((rows, 1), dtype=torch.float32, device="cuda") for _ in range(count)]
xs = [torch.from_numpy(orc.bench_input_array(cols, 1, i)).cuda() for i in range(count)]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for it in range(6):
        if staged:
            cg.gemm_stages(sets[it % 2], xs, ys, list(range(count)), stream=s)
        else:
            cg.gemm_group(sets[it % 2], xs, stream=s)
s.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
lib = _lib.load()
lib.cg_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
bufs = []
for k in range(2):
    buf = np.zeros(sms * 64, dtype=np.uint64)
    _lib.check(lib.cg_debug_stamps(sets[k][0].handle, buf.ctypes.data, sms * 64))
    bufs.append(buf.reshape(sms, 64).astype(np.int64))
prev, st = bufs[0], bufs[1]  # launch 4 (set 0) then launch 5 (set 1)
valid = st[:, 0] > 0
t0 = st[valid, 0].min()
print(sets[0][0].info)
pend = prev[prev[:, 63] > 0, 63]
print(f"previous launch: last CTA end {(pend.max() - t0) / 1e3:7.2f} us (rel. to this launch's first start)")


def show(name, col):
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1000.0
        print(f"{name:18s} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")


show("pdl_wait passed", st[valid, 62])
names = [(0, "start"), (7, "synced"), (4, "inputs ok"), (5, "x staged"), (6, "built"),
         (1, "gathered"), (2, "zero barrier ok"), (3, "task end")]
for k in range(min(count, 3)):
    for slot, nm in names:
        show(f"task{k} {nm}", st[valid, k * 8 + slot])
for slot, nm in ((48, "barrier entered"), (49, "bulk drained"), (50, "arrived"), (51, "released")):
    show(nm, st[valid, slot])
show("kernel end", st[valid, 63])
