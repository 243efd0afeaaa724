"""CGMM container fixtures written by the REFERENCE serializer (storage.py), for the loader tests.

Run in the authoring container (imports /root/reference); writes tests/golden/cgmm/*.cgmm and
tests/golden/cgmm_planes.npz (the reference-decoded code planes, scales, codebooks).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
from codegemm import quantizer, storage  # noqa: E402

CASES = [("m1v4b8g128", 48, 512, dict(v=4, m=1, b=8, g=128)),
         ("m2v8b8g128", 40, 1024, dict(v=8, m=2, b=8, g=128)),
         ("m1v4b3grow", 37, 200, dict(v=4, m=1, b=3, g=-1)),
         ("m2v4b6g64", 33, 256, dict(v=4, m=2, b=6, g=64))]
out_dir = os.path.join(ROOT, "tests", "golden", "cgmm")
os.makedirs(out_dir, exist_ok=True)
arrays = {}
for name, rows, cols, kw in CASES:
    q = quantizer.random_layer(rows, cols, quantizer.QuantConfig(**kw), seed=rows * 131 + cols)
    path = os.path.join(out_dir, name + ".cgmm")
    storage.serialize(q, path)
    back = storage.deserialize(path)
    for t, p in enumerate(back.planes):
        arrays[f"{name}/codes{t}"] = p.codes
    for t, b in enumerate(back.books):
        arrays[f"{name}/book{t}"] = b.entries
    arrays[f"{name}/scales"] = back.scales.scales
    print(name, os.path.getsize(path), "bytes")
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cgmm_planes.npz"), **arrays)
