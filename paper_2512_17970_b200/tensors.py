"""binary16 activation container (the reference's ``Matrix``).

Mirrors ``/root/reference/pkg/src/codegemm/tensors.py:81-143``: a read-only,
row-major, little-endian float16 array; ``widened()`` is the exact binary32
view every consumer computes with.  For the decode path X is (K, N): one
column per token.
"""

from __future__ import annotations

import numpy as np

from .errors import ShapeError

_F16 = np.dtype("<f2")
_QNAN = 0x7E00


def encode_f16_array(values) -> np.ndarray:
    """Round to binary16 (nearest-even), returning uint16 bit patterns.

    NaNs become the canonical quiet NaN 0x7E00 (tensors.py:47-58).
    """
    src = np.asarray(values, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        out = src.astype(_F16).view(np.uint16).copy()
    nan = np.isnan(src)
    if nan.any():
        out[nan] = _QNAN
    return out


class Matrix:
    """Immutable 2-D binary16 matrix."""

    __slots__ = ("_data", "__weakref__")

    def __init__(self, data: np.ndarray, copy: bool = True):
        arr = np.asarray(data)
        if arr.ndim != 2:
            raise ShapeError(f"matrix must be 2-D, got ndim={arr.ndim}")
        if min(arr.shape) < 1:
            raise ShapeError(f"matrix dims must be >= 1, got {arr.shape}")
        if arr.dtype != _F16:
            raise ShapeError(f"matrix data must be little-endian float16, got {arr.dtype}")
        arr = np.array(arr, copy=True) if copy else np.ascontiguousarray(arr)
        arr.flags.writeable = False
        self._data = arr

    @classmethod
    def from_array(cls, values) -> "Matrix":
        src = np.asarray(values, dtype=np.float64)
        if src.ndim != 2:
            raise ShapeError(f"matrix must be 2-D, got ndim={src.ndim}")
        return cls(encode_f16_array(src).view(_F16), copy=False)

    @property
    def rows(self) -> int:
        return int(self._data.shape[0])

    @property
    def cols(self) -> int:
        return int(self._data.shape[1])

    @property
    def data(self) -> np.ndarray:
        return self._data

    @property
    def bits(self) -> np.ndarray:
        return self._data.view(np.uint16)

    def widened(self, dtype=np.float32) -> np.ndarray:
        return self._data.astype(dtype)

    def bit_equal(self, other: "Matrix") -> bool:
        return self._data.shape == other.data.shape and bool(
            np.array_equal(self.bits, np.asarray(other.data).view(np.uint16))
        )

    def __repr__(self) -> str:
        return f"Matrix(rows={self.rows}, cols={self.cols})"
