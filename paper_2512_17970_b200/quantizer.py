"""The quantized-layer format the decode path consumes.

These containers restate the operator-API tensor layout of the reference
(``/root/reference/pkg/src/codegemm/quantizer.py``):

* ``QuantConfig``     (v, m, b, g, seed, kmeans_iters) with the same validation
                      rules (quantizer.py:35-84)
* ``Codebook``        (2**b, v) binary16 centroids (quantizer.py:87-113)
* ``ScalePlane``      (rows, cols/g_eff) binary16, > 0 (quantizer.py:116-132)
* ``CodePlane``       (rows, cols/v) uint16 code indices (quantizer.py:135-145)
* ``QuantizedLayer``  container + invariants, ``segment_groups`` (quantizer.py:148-226)
* ``pack_codes`` / ``unpack_codes``  LSB-first b-bit stream (quantizer.py:471-497)
* ``random_layer``    the seeded synthetic generator (quantizer.py:500-523),
                      bit-identical draws so CPU and GPU see the same layer

The engines accept these objects or the reference's own (duck-typed on the
same attribute names).  The offline k-means quantizer is outside the decode
path and is not part of this package.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, IntegrityError

_F16 = np.dtype("<f2")


@dataclass(frozen=True)
class QuantConfig:
    v: int
    m: int
    b: int
    g: int = -1
    seed: int = 0
    kmeans_iters: int = 25

    def __post_init__(self):
        checks = (
            (self.v >= 1, f"v must be >= 1, got {self.v}"),
            (self.m >= 1, f"m must be >= 1, got {self.m}"),
            (1 <= self.b <= 16, f"b must be in [1, 16], got {self.b}"),
            (self.g == -1 or self.g >= self.v, f"g must be >= v (got g={self.g}, v={self.v})"),
            (self.g == -1 or self.g % self.v == 0,
             f"g must be a multiple of v (got g={self.g}, v={self.v})"),
            (0 <= self.seed < 2**64, "seed must fit in 64 bits"),
            (self.kmeans_iters >= 1, "kmeans_iters must be >= 1"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)

    def group_size_for(self, cols: int) -> int:
        return cols if self.g == -1 else self.g

    def validate_shape(self, rows: int, cols: int) -> None:
        if rows < 1 or cols < 1:
            raise ConfigError(f"matrix dims must be >= 1, got {rows}x{cols}")
        if cols % self.v:
            raise ConfigError(f"cols={cols} not divisible by v={self.v}")
        if cols % self.group_size_for(cols):
            raise ConfigError(f"cols={cols} not divisible by g={self.g}")


def _frozen(arr: np.ndarray) -> np.ndarray:
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class Codebook:
    entries: np.ndarray  # (2**b, v) float16

    def __post_init__(self):
        e = self.entries
        if e.ndim != 2 or e.dtype != _F16:
            raise IntegrityError("codebook entries must be a 2-D float16 array")
        k = e.shape[0]
        if k < 2 or (k & (k - 1)):
            raise IntegrityError(f"codebook entry count {k} is not a power of two >= 2")
        if not np.isfinite(e.astype(np.float32)).all():
            raise IntegrityError("codebook entries must be finite")
        _frozen(e)

    @property
    def size(self) -> int:
        return int(self.entries.shape[0])

    @property
    def vector_len(self) -> int:
        return int(self.entries.shape[1])

    def widened(self) -> np.ndarray:
        return self.entries.astype(np.float32)


@dataclass(frozen=True)
class ScalePlane:
    scales: np.ndarray  # (rows, groups) float16

    def __post_init__(self):
        s = self.scales
        if s.ndim != 2 or s.dtype != _F16:
            raise IntegrityError("scales must be a 2-D float16 array")
        w = s.astype(np.float32)
        if not (np.isfinite(w).all() and (w > 0.0).all()):
            raise IntegrityError("scales must be finite and strictly positive")
        _frozen(s)

    def widened(self) -> np.ndarray:
        return self.scales.astype(np.float32)


@dataclass(frozen=True)
class CodePlane:
    codes: np.ndarray  # (rows, segments) uint16

    def __post_init__(self):
        c = self.codes
        if c.ndim != 2 or c.dtype != np.uint16:
            raise IntegrityError("codes must be a 2-D uint16 array")
        _frozen(c)


@dataclass(frozen=True, eq=False)
class QuantizedLayer:
    rows: int
    cols: int
    config: QuantConfig
    scales: ScalePlane
    planes: tuple
    books: tuple

    def __post_init__(self):
        cfg = self.config
        cfg.validate_shape(self.rows, self.cols)
        if len(self.planes) != cfg.m or len(self.books) != cfg.m:
            raise IntegrityError(
                f"expected {cfg.m} planes and books, got "
                f"{len(self.planes)} planes / {len(self.books)} books"
            )
        want_scales = (self.rows, self.groups)
        if self.scales.scales.shape != want_scales:
            raise IntegrityError(f"scales shape {self.scales.scales.shape} != {want_scales}")
        for plane in self.planes:
            if plane.codes.shape != (self.rows, self.segments):
                raise IntegrityError(
                    f"plane shape {plane.codes.shape} != {(self.rows, self.segments)}"
                )
            if plane.codes.max(initial=0) >= 2**cfg.b:
                raise IntegrityError(f"code out of range for b={cfg.b}")
        for book in self.books:
            if book.entries.shape != (2**cfg.b, cfg.v):
                raise IntegrityError(
                    f"codebook shape {book.entries.shape} != {(2 ** cfg.b, cfg.v)}"
                )

    @property
    def segments(self) -> int:
        return self.cols // self.config.v

    @property
    def groups(self) -> int:
        return self.cols // self.config.group_size_for(self.cols)

    def segment_groups(self) -> np.ndarray:
        g_eff = self.config.group_size_for(self.cols)
        return (np.arange(self.segments) * self.config.v) // g_eff


def pack_codes(plane, b: int) -> bytes:
    """Code i occupies stream bits [i*b, (i+1)*b), LSB first, byte padded."""
    if not 1 <= b <= 16:
        raise ConfigError(f"b must be in [1, 16], got {b}")
    flat = np.asarray(getattr(plane, "codes", plane)).reshape(-1).astype(np.uint32)
    if flat.size and int(flat.max()) >= (1 << b):
        raise ValueError(f"code {int(flat.max())} out of range for b={b}")
    bitplanes = (flat[:, None] >> np.arange(b, dtype=np.uint32)) & 1
    return np.packbits(bitplanes.astype(np.uint8).ravel(), bitorder="little").tobytes()


def unpack_codes(data: bytes, rows: int, segments: int, b: int) -> CodePlane:
    if not 1 <= b <= 16:
        raise ConfigError(f"b must be in [1, 16], got {b}")
    count = rows * segments
    need = (count * b + 7) // 8
    if len(data) < need:
        raise ValueError(f"packed stream too short: {len(data)} < {need} bytes")
    bits = np.unpackbits(np.frombuffer(data, np.uint8, count=need), bitorder="little")
    weights = np.left_shift(np.uint32(1), np.arange(b, dtype=np.uint32))
    vals = bits[: count * b].reshape(count, b).astype(np.uint32) @ weights
    return CodePlane(vals.astype(np.uint16).reshape(rows, segments))


def random_layer(rows: int, cols: int, cfg: QuantConfig, seed=None) -> QuantizedLayer:
    """Seeded synthetic layer; same draw order as quantizer.py:513-522.

    scales |N(0,1)|*0.25 + 0.5, then m codebooks N(0,1)*0.5, then m uniform
    code planes, all from one ``default_rng(seed)`` stream.
    """
    cfg.validate_shape(rows, cols)
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    k = 1 << cfg.b
    groups = cols // cfg.group_size_for(cols)
    scale_draw = np.abs(rng.standard_normal((rows, groups))) * 0.25 + 0.5
    books = tuple(Codebook((rng.standard_normal((k, cfg.v)) * 0.5).astype(_F16))
                  for _ in range(cfg.m))
    planes = tuple(CodePlane(rng.integers(0, k, size=(rows, cols // cfg.v), dtype=np.uint16))
                   for _ in range(cfg.m))
    return QuantizedLayer(rows, cols, cfg, ScalePlane(scale_draw.astype(_F16)), planes, books)
