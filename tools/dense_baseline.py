"""GPU baselines for the same Llama-3-8B decoder block (the paper's A.4
comparison): dense binary16 weights through cuBLAS (torch.matmul), and a naive dequantize
(codes -> binary16 W by gather, per-group scales) + cuBLAS per call.  Weights rotated over
copies larger than L2, CUDA graphs, CUDA-event timing.  Prints one JSON line.

python tools/dense_baseline.py [batch]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec = bench.block_spec("8b")
dev = torch.device("cuda")
l2 = torch.cuda.get_device_properties(0).L2_cache_size
dense_bytes = sum(2 * r * c for _, r, c in spec)
copies = max(2, int(np.ceil(3 * l2 / dense_bytes)))
g = torch.Generator(device="cuda").manual_seed(0)
W = [[torch.randn((r, c), device=dev, dtype=torch.float16, generator=g) * 0.02 for _, r, c in spec]
     for _ in range(copies)]
X = [torch.randn((c, n), device=dev, dtype=torch.float16, generator=g) for _, r, c in spec]


def timed(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    s.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        fn()
    with torch.cuda.stream(s):
        for _ in range(3):
            gr.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            gr.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def dense_step():
    for k in range(copies):
        for w, x in zip(W[k], X):
            torch.matmul(w, x)


us_dense = timed(dense_step) / copies
del W
torch.cuda.empty_cache()

# naive dequant + cuBLAS: m1v4g128 codes (uint8), codebook (256, 4) fp16, scales (rows, cols/128)
cfg = bench.CONFIGS["m1v4g128"]
Q = []
for k in range(copies):
    layers = []
    for _, r, c in spec:
        codes = torch.randint(0, 256, (r, c // 4), device=dev, dtype=torch.uint8, generator=g)
        book = (torch.randn((256, 4), device=dev, generator=g) * 0.5).half()
        scales = (torch.rand((r, c // 128), device=dev, generator=g) + 0.5).half()
        layers.append((codes, book, scales))
    Q.append(layers)


def dequant_step():
    for k in range(copies):
        for (codes, book, scales), x in zip(Q[k], X):
            r = codes.shape[0]
            w = book[codes.long()].reshape(r, -1)                       # (r, c) binary16
            w = (w.view(r, -1, 128) * scales.unsqueeze(-1)).reshape(r, -1)
            torch.matmul(w, x)


us_deq = timed(dequant_step, reps=10) / copies
code_bytes = sum(bench.layer_bytes(r, c, cfg, n) for _, r, c in spec)
print(json.dumps({
    "workload": f"llama8b decoder-block linears (reference suite), batch {n}",
    "dense_fp16_cublas": {"us_per_block": round(us_dense, 2),
                          "GBps": round((dense_bytes + sum(2 * c * n + 2 * r * n for _, r, c in spec))
                                        / (us_dense * 1e-6) / 1e9, 1),
                          "weight_bytes": dense_bytes},
    "dequant_then_cublas": {"us_per_block": round(us_deq, 2),
                            "note": "torch gather dequant of m1v4g128 codes + per-group scales, then cuBLAS"},
    "codegemm_weight_bytes": code_bytes,
}), flush=True)
