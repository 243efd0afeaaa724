"""Per-task phase timeline of the staged decoder-block launch (diagnostics).

python tools/stamps_block.py [CHAIN]   -- bench.py's N=1 step, CHAIN blocks chained per launch
(u=2, q->o->gate/up->down, the next block's q,k,v reading y_down).  A graph of two such launches
(different weights) is replayed; the stamps of the second, in us from its first task start.
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

chain = int(sys.argv[1]) if len(sys.argv) > 1 else 1
INDEP = int(os.environ.get("INDEP", "0"))  # 1: every layer independent, one stage
XCHG = int(os.environ.get("XCHG", "0"))  # 1: through a world-1 comm, every layer pushed
cfg = bench.CONFIGS["m1v4g128"]
spec = bench.block_spec("8b")
nl = len(spec)
sets = []
for k in range(2):
    layers = [cg.DeviceLayer(bench.make_layer(r, c, cfg, 100 * k + 7 * j + i), u=bench.TILING_U or 4)
              for j in range(chain) for i, (_, r, c) in enumerate(spec)]
    if XCHG:
        from paper_2512_17970_b200 import dist as cgd
        glay = cgd.GatheredLayout([r for j in range(chain) for (_, r, c) in spec], 1, 1)
        comm = cgd.PeerExchange(1, 0, glay.nbytes, timeout_ms=20000)
        ys = [glay.gathered(comm, i) for i in range(chain * nl)]
    else:
        comm = None
        ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for j in range(chain)
              for (_, r, c) in spec]
    x0 = torch.from_numpy(orc.bench_input_array(spec[0][2], 1, k)).cuda()
    xs, st = [], []
    for j in range(chain):
        for i, src in enumerate(bench.STEP_XSRC):
            if src is not None:
                xs.append(ys[j * nl + src])
            else:
                xs.append(x0 if j == 0 else ys[(j - 1) * nl + nl - 1])
            st.append(4 * j + bench.STEP_STAGES[i])
    if INDEP:
        xs = [torch.from_numpy(orc.bench_input_array(c, 1, 10 * k + i)).cuda()
              for j in range(chain) for i, (_, r, c) in enumerate(spec)]
        st = [0] * len(layers)
    sets.append((layers, xs, ys, st, comm))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for L, xs, ys, st, cm in sets:
        cg.gemm_stages(L, xs, ys, st, stream=s, comm=cm, xchg=[1] * len(L) if cm else None)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for L, xs, ys, st, cm in sets:
        cg.gemm_stages(L, xs, ys, st, stream=s, comm=cm, xchg=[1] * len(L) if cm else None)
with torch.cuda.stream(s):
    for _ in range(3):
        g.replay()
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
lib = _lib.load()
lib.cg_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
bufs = []
for k in range(2):
    b = np.zeros(sms * 128, dtype=np.uint64)
    _lib.check(lib.cg_debug_stamps(sets[k][0][0].handle, b.ctypes.data, sms * 128))
    bufs.append(b.reshape(sms, 128).astype(np.int64))
pv, st = bufs
t0 = st[st[:, 0] > 0, 0].min()
print(f"chain {chain}: previous launch (same graph): last kernel end {(pv[:, 127].max() - t0) / 1e3:.2f} us")


def show(name, col):
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1000.0
        print(f"{name:22s} n={len(col):3d} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")


show("kernel entry", st[:, 124])
show("table copied", st[:, 88])
show("first task located", st[:, 89])
show("weights issued", st[:, 90])
show("before pdl_wait (t0)", st[:, 91])
show("pdl_wait passed", st[:, 126])
show("x issued", st[:, 92])
show("zeroing done (tid 0)", st[:, 93])
show("prologue done", st[:, 125])
names = [(0, "start"), (7, "synced"), (4, "inputs ok"), (5, "x staged"), (6, "table ready"),
         (1, "gathered"), (2, "zero ok/flush"), (3, "task end")]
for k in range(11):
    for slot, nm in names:
        if slot in (0, 7, 4, 5, 6, 1, 3):
            show(f"task{k} {nm}", st[:, k * 8 + slot])
for b in range(7):
    for j, nm in enumerate(("entered", "drained", "arrived", "released")):
        show(f"barrier{b} {nm}", st[:, 96 + 4 * b + j])
for b in range(4):
    show(f"xchg{b} pushed", st[:, 112 + 2 * b])
    show(f"xchg{b} all arrived", st[:, 113 + 2 * b])
show("kernel end", st[:, 127])
if os.environ.get("GRAN"):  # timer granularity: gcd of the stamp offsets
    v = st[st > 0] - t0
    print("stamp granularity (ns):", int(np.gcd.reduce(v[v > 0].astype(np.int64))),
          "sample offsets:", sorted(set((v % 1000).tolist()))[:12])
if os.environ.get("FINE"):
    for w in range(16):
        show(f"task1 warp{w:2d} at post-build barrier", st[:, 96 + w])
    for k, nm in enumerate(("loop top", "stages passed", "before run_task", "tiles issued", "x loaded")):
        show(f"task1 fine {nm}", st[:, 112 + k])
