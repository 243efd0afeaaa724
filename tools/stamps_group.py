"""Per-task phase timeline of a grouped launch (diagnostics; CG_STAMPS=1).

python tools/stamps_group.py ROWS COLS COUNT
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
layers = [cg.DeviceLayer(cg.random_layer(rows, cols, cg.QuantConfig(v=4, m=1, b=8, g=128),
                                         seed=i)) for i in range(count)]
xs = [torch.from_numpy(orc.bench_input_array(cols, 1, i)).cuda() for i in range(count)]
for _ in range(3):
    cg.gemm_group(layers, xs)
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
buf = np.zeros(sms * 32, dtype=np.uint64)
lib = _lib.load()
lib.cg_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
_lib.check(lib.cg_debug_stamps(layers[0].handle, buf.ctypes.data, sms * 32))
st = buf.reshape(sms, 4, 8).astype(np.int64)
valid = st[:, 0, 0] > 0
st = st[valid]
t0 = st[:, 0, 0].min()
print(layers[0].info)
names = {0: "start", 7: "synced", 4: "mbar ok", 1: "books cvt", 5: "x staged", 6: "built",
         2: "issued", 3: "gathered"}
for k in range(min(count, 3)):
    for slot, nm in names.items():
        col = st[:, k, slot]
        col = col[col > 0]
        if len(col):
            r = (col - t0) / 1000.0
            print(f"task{k} {nm:9s} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")
end = (st[:, 3, 7] - t0) / 1000.0
print(f"kernel end   min {end.min():7.2f} med {np.median(end):7.2f} max {end.max():7.2f}")
