"""The C-ABI library: loads, exports every declared symbol, fails loudly.

CPU-only checks (no compute calls need a GPU).
"""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2512_17970_b200 import _lib
from helpers import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "codegemm_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_binding():
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cg_[a-z0-9_]+)\b", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_abi_version_and_error_mapping():
    lib = _lib.load()
    assert lib.cg_abi_version() == 1
    rc = lib.cg_layer_create(None, None, None, 1, 1, 1, 1, 1, -1, None, ctypes.byref(ctypes.c_void_p()))
    assert rc == _lib.CG_ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(rc)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu():
    import numpy as np

    import paper_2512_17970_b200 as cg

    assert _lib.load().cg_device_count() == 0
    layer = cg.random_layer(16, 64, cg.QuantConfig(v=4, m=1, b=8, g=32), seed=0)
    with pytest.raises(cg.CudaError):
        cg.codegemm_gemm(layer, cg.Matrix.from_array(np.ones((64, 1))))


def test_config_errors_map_to_reference_classes():
    import numpy as np

    import paper_2512_17970_b200 as cg

    lib = _lib.load()
    codes = np.zeros((2, 3), np.uint16)
    books = np.zeros((4, 2), np.uint16)
    scales = np.ones((2, 1), np.uint16)
    ptrs = (ctypes.c_void_p * 1)(codes.ctypes.data)
    bptrs = (ctypes.c_void_p * 1)(books.ctypes.data)
    h = ctypes.c_void_p()
    # cols=6 with v=4: not divisible -> ConfigError before any device use
    rc = lib.cg_layer_create(ptrs, bptrs, scales.ctypes.data, 2, 6, 4, 1, 2, -1, None,
                             ctypes.byref(h))
    assert rc == _lib.CG_ERR_CONFIG
    with pytest.raises(cg.ConfigError):
        _lib.check(rc)
