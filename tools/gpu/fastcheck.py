"""Which golden small cases have a fused-kernel plan (diagnostics)."""
import os
import sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import conftest  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from helpers import layer_from_case  # noqa: E402

for c in conftest._cases("small_layers.npz"):
    dl = cg.DeviceLayer(layer_from_case(c))
    print(c["name"], c["v"], c["m"], c["b"], c["g"], c["n"], dl.info["fast_supported"], dl.info["u"])
