"""ctypes wrapper of oracle/_build/libcg_oracle.so (test infrastructure only).

Builds the C restatement on first use with the committed Makefile (gcc).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libcg_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        vp, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        lib.cgo_codegemm.argtypes = [vp, vp, vp, vp, i64, i64, i, i, i, i64, i, i, i, vp]
        lib.cgo_codegemm.restype = i
        lib.cgo_psum_tables.argtypes = [vp, vp, i, i, i, i64, i, vp]
        lib.cgo_psum_tables.restype = i
        _lib = lib
    return _lib


def _ptrs(arrays):
    return (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])


def codegemm(codes, books, scales, x, v, g, t_w=32, threads=1) -> np.ndarray:
    """Bit-identical to the reference codegemm_gemm (see cg_oracle.c)."""
    codes = [np.ascontiguousarray(c, dtype=np.uint16) for c in codes]
    books = [np.ascontiguousarray(np.asarray(b).view(np.uint16)) for b in books]
    scales = np.ascontiguousarray(np.asarray(scales).view(np.uint16))
    x = np.ascontiguousarray(np.asarray(x).view(np.uint16))
    rows, segs = codes[0].shape
    cols = segs * v
    n = x.shape[1]
    b = int(books[0].shape[0]).bit_length() - 1
    y = np.empty((rows, n), dtype=np.float32)
    rc = load().cgo_codegemm(_ptrs(codes), _ptrs(books), scales.ctypes.data, x.ctypes.data,
                             rows, cols, v, len(codes), b, g, n, t_w, threads, y.ctypes.data)
    if rc:
        raise ValueError("cgo_codegemm rejected its arguments")
    return y


def psum_tables(books, x, v) -> np.ndarray:
    books = [np.ascontiguousarray(np.asarray(b).view(np.uint16)) for b in books]
    x = np.ascontiguousarray(np.asarray(x).view(np.uint16))
    k_len, n = x.shape
    kcount = books[0].shape[0]
    out = np.empty((len(books), k_len // v, kcount, n), dtype=np.float32)
    rc = load().cgo_psum_tables(_ptrs(books), x.ctypes.data, len(books),
                                int(kcount).bit_length() - 1, v, k_len, n, out.ctypes.data)
    if rc:
        raise ValueError("cgo_psum_tables rejected its arguments")
    return out
