import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def _cases(fname):
    with np.load(os.path.join(GOLDEN, fname), allow_pickle=False) as z:
        data = {k: z[k] for k in z.files}
    out = []
    for name in data["names"]:
        p = f"{name}/"
        case = {k[len(p):]: v for k, v in data.items() if k.startswith(p)}
        case["name"] = str(name)
        meta = case["meta"]
        case["rows"], case["cols"], case["v"], case["m"], case["b"], case["g"], case["n"] = (
            int(x) for x in meta[:7])
        case["codes"] = [case[f"codes{t}"] for t in range(case["m"])]
        case["books"] = [case[f"book{t}"] for t in range(case["m"])]
        out.append(case)
    return out


@pytest.fixture(scope="session")
def small_cases():
    return _cases("small_layers.npz")


@pytest.fixture(scope="session")
def sweep_cases():
    return _cases("quantized_sweep.npz")


@pytest.fixture(scope="session")
def kat():
    with np.load(os.path.join(GOLDEN, "kat.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def bench_golden():
    with np.load(os.path.join(GOLDEN, "bench_shapes.npz")) as z:
        return {k: z[k] for k in z.files}
