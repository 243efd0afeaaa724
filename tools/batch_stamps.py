"""Per-CTA timeline of one batch-kernel launch (diagnostics, CG_STAMPS=1).

python tools/batch_stamps.py ROWS COLS N
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

rows, cols, n = (int(a) for a in sys.argv[1:4])
dl = cg.DeviceLayer(bench.make_layer(rows, cols, bench.CONFIGS["m1v4g128"], 5))
x = torch.from_numpy(orc.bench_input_array(cols, n, 1)).cuda()
y = torch.empty((rows, n), dtype=torch.float32, device="cuda")
for _ in range(3):
    dl.gemm(x, y)
torch.cuda.synchronize()
buf = np.zeros(64 * 1024, dtype=np.uint64)
lib = _lib.load()
lib.cg_debug_batch_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int64]
_lib.check(lib.cg_debug_batch_stamps(buf.ctypes.data, buf.size))
st = buf.reshape(1024, 64)[:148].astype(np.int64)
t0 = st[:, 0].min()
names = {0: "start", 1: "table+x staged"}
for i in range(2, 20):
    names[i] = f"task{(i - 2) // 3} " + ["issued/wait", "data in", "done"][(i - 2) % 3]
for i in range(40, 44):
    names[i] = f"task{i - 40} before issue"
for i in range(50, 54):
    names[i] = f"task{i - 50} loop top"
for i in list(range(20)) + list(range(40, 44)) + list(range(50, 54)):
    v = st[:, i]
    v = v[v > 0]
    if len(v) == 0:
        continue
    v = (v - t0) / 1e3
    print(f"{names[i]:18s} n={len(v):3d} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
