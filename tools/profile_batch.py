"""One batch-kernel call under a profiler: python tools/profile_batch.py ROWS COLS N [config]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402

rows, cols, n = (int(a) for a in sys.argv[1:4])
cfg = bench.CONFIGS[sys.argv[4] if len(sys.argv) > 4 else "m1v4g128"]
dl = cg.DeviceLayer(bench.make_layer(rows, cols, cfg, 5))
x = torch.from_numpy(orc.bench_input_array(cols, n, 1)).cuda()
y = torch.empty((rows, n), dtype=torch.float32, device="cuda")
for _ in range(5):
    dl.gemm(x, y)
torch.cuda.synchronize()
print("ok", dl.query()["batch_ready"])
