"""Per-CTA phase timeline of the fused kernel (diagnostics; CG_STAMPS=1)."""
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

rows, cols = int(sys.argv[1]), int(sys.argv[2])
u = int(sys.argv[3]) if len(sys.argv) > 3 else 0
q = cg.random_layer(rows, cols, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=1)
dl = cg.DeviceLayer(q, u=u)
x = torch.from_numpy(orc.bench_input_array(cols, 1, 0)).cuda()
for _ in range(3):
    y = dl.gemm(x)
torch.cuda.synchronize()
n = dl.info["n_tasks"]
buf = np.zeros(n * 8, dtype=np.uint64)
lib = _lib.load()
lib.cg_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
_lib.check(lib.cg_debug_stamps(dl.handle, buf.ctypes.data, n * 8))
st = buf.reshape(n, 8).astype(np.int64)
t0 = st[:, 0].min()
rel = (st - t0) / 1000.0  # us
names = ["start", "loads+fixups", "built", "gathered", "end", "x staged"]
print(dl.info)
for k, nm in enumerate(names):
    col = rel[:, k]
    col = col[st[:, k] > 0]
    if len(col):
        print(f"{nm:16s} min {col.min():7.2f}  median {np.median(col):7.2f}  max {col.max():7.2f} us")
d = rel[:, 3] - rel[:, 2]
print(f"gather duration: min {d.min():.2f} median {np.median(d):.2f} max {d.max():.2f} us")
d = rel[:, 2] - rel[:, 5]
print(f"build only: min {d.min():.2f} median {np.median(d):.2f} max {d.max():.2f} us")
d = rel[:, 5] - rel[:, 1]
print(f"x wait: min {d.min():.2f} median {np.median(d):.2f} max {d.max():.2f} us")
d = rel[:, 2] - rel[:, 1]
print(f"build duration: min {d.min():.2f} median {np.median(d):.2f} max {d.max():.2f} us")
d = rel[:, 1] - rel[:, 0]
print(f"prologue duration: min {d.min():.2f} median {np.median(d):.2f} max {d.max():.2f} us")
