"""CPU oracle for the CodeGEMM decode path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy over plain arrays, the reference
algorithm that the B200 kernels replace.  It is the *checker*: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import it.  The product path (``paper_2512_17970_b200``) never imports,
links or calls anything under ``oracle/`` and fails loudly when its CUDA
library is missing.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks every function
here against golden vectors produced by the reference package itself
(``oracle/make_golden.py`` imports ``/root/reference/pkg/src/codegemm`` in the
authoring container and writes ``tests/golden/*.npz``), plus the reference's
own known-answer tests (``pkg/tests/test_engines.py:86-108``).

Citations are ``file:line`` into ``/root/reference/pkg/src/codegemm/``.

Arrays used throughout (the reference's operator layout):

* ``codes``  -- list of m uint16 arrays (rows, K/v)     (quantizer.py:135-145)
* ``books``  -- list of m float16 arrays (2**b, v)       (quantizer.py:87-113)
* ``scales`` -- float16 array (rows, K/g_eff)            (quantizer.py:116-132)
* ``x``      -- float16 array (K, N), one column/token   (tensors.py:81-103)
"""

from __future__ import annotations

import numpy as np

F16 = np.dtype("<f2")


# --------------------------------------------------------------------------
# synthetic inputs (bit-identical generators)
# --------------------------------------------------------------------------

def group_size(cols: int, g: int) -> int:
    """g_eff: g, or the whole row when g == -1 (quantizer.py:72-74)."""
    return cols if g == -1 else g


def random_layer_arrays(rows: int, cols: int, v: int, m: int, b: int, g: int, seed: int):
    """Draw (scales, books, codes) in the reference order (quantizer.py:500-523).

    One ``default_rng(seed)`` stream: scales |N(0,1)|*0.25+0.5 -> f16, then the
    m codebooks N(0,1)*0.5 -> f16, then the m code planes uniform in [0, 2**b).
    """
    rng = np.random.default_rng(seed)
    k = 1 << b
    segs = cols // v
    groups = cols // group_size(cols, g)
    scales = (np.abs(rng.standard_normal((rows, groups))) * 0.25 + 0.5).astype(F16)
    books = [(rng.standard_normal((k, v)) * 0.5).astype(F16) for _ in range(m)]
    codes = [rng.integers(0, k, size=(rows, segs), dtype=np.uint16) for _ in range(m)]
    return scales, books, codes


def bench_input_array(k_in: int, m_batch: int, seed: int = 0) -> np.ndarray:
    """Seeded Gaussian activations (K, batch) in f16 (bench.py:162-165)."""
    rng = np.random.default_rng((seed, k_in, m_batch, 0x1A))
    return rng.standard_normal((k_in, m_batch)).astype(F16)


def bench_layer_seed(n_out: int, k_in: int, seed: int = 0) -> int:
    """Layer seed used by bench_layer: seed ^ N ^ K (bench.py:168-170)."""
    return seed ^ n_out ^ k_in


# --------------------------------------------------------------------------
# Psumbook build (engines.py:115-134)
# --------------------------------------------------------------------------

def psum_tables(books32, x32: np.ndarray, v: int) -> np.ndarray:
    """(m, segs, 2**b, n) float32 table of centroid . segment dot products.

    Each entry starts at +0.0 and adds the products c[i,k]*x[j*v+k] for k
    ascending, one binary32 rounding per add (engines.py:126-133).  Products
    of f16-widened values are exact in binary32, so the only roundings are
    the adds.
    """
    x32 = np.asarray(x32, dtype=np.float32)
    width, n = x32.shape
    segs = width // v
    m = len(books32)
    k = books32[0].shape[0]
    out = np.zeros((m, segs, k, n), dtype=np.float32)
    for t in range(m):
        c = np.asarray(books32[t], dtype=np.float32)
        for j in range(segs):
            acc = out[t, j]
            for kk in range(v):
                acc += c[:, kk:kk + 1] * x32[j * v + kk][None, :]
    return out


def segment_groups(cols: int, v: int, g: int) -> np.ndarray:
    """Scale column of every segment: (seg*v)//g_eff (quantizer.py:195-199)."""
    return (np.arange(cols // v) * v) // group_size(cols, g)


def tile_spans(k_len: int, t_w: int):
    """Ascending (start, width) K-tiles, last one partial (engines.py:234-242)."""
    return [(s, min(t_w, k_len - s)) for s in range(0, k_len, t_w)]


# --------------------------------------------------------------------------
# engines
# --------------------------------------------------------------------------

def codegemm(codes, books, scales, x, v: int, g: int, t_w: int = 32, t_h: int = 2048):
    """Lookup-table GEMM, bit-identical to the reference codegemm_gemm.

    Follows engines.py:245-316: per K-tile build the tables for all columns
    (engines.py:298-299), then per row block gather by code, sum the m
    codebooks (t ascending) into seg_sum, and add scale*seg_sum into the
    single running accumulator (engines.py:286-294).  Returns float32
    (rows, N).
    """
    m = len(codes)
    rows, segs = codes[0].shape
    cols = segs * v
    x32 = np.asarray(x).astype(np.float32)
    books32 = [np.asarray(bk).astype(np.float32) for bk in books]
    scales32 = np.asarray(scales).astype(np.float32)
    sg = segment_groups(cols, v, g)
    n = x32.shape[1]
    y = np.zeros((rows, n), dtype=np.float32)
    blocks = [(r0, min(r0 + t_h, rows)) for r0 in range(0, rows, t_h)]
    for start, width in tile_spans(cols, t_w):
        tables = psum_tables(books32, x32[start:start + width], v)
        seg0 = start // v
        for r0, r1 in blocks:
            for j in range(tables.shape[1]):
                seg = seg0 + j
                seg_sum = np.zeros((r1 - r0, n), dtype=np.float32)
                for t in range(m):
                    seg_sum += tables[t, j][codes[t][r0:r1, seg]]
                y[r0:r1] += scales32[r0:r1, sg[seg]][:, None] * seg_sum
    return y


def dequant_mirrored(codes, books, scales, x, v: int, g: int):
    """The bit-exact twin without tables (engines.py:211-231)."""
    m = len(codes)
    rows, segs = codes[0].shape
    cols = segs * v
    x32 = np.asarray(x).astype(np.float32)
    books32 = [np.asarray(bk).astype(np.float32) for bk in books]
    scales32 = np.asarray(scales).astype(np.float32)
    sg = segment_groups(cols, v, g)
    n = x32.shape[1]
    y = np.zeros((rows, n), dtype=np.float32)
    for seg in range(segs):
        base = seg * v
        seg_sum = np.zeros((rows, n), dtype=np.float32)
        for t in range(m):
            chosen = books32[t][codes[t][:, seg]]
            psum = np.zeros((rows, n), dtype=np.float32)
            for kk in range(v):
                psum += chosen[:, kk:kk + 1] * x32[base + kk][None, :]
            seg_sum += psum
        y += scales32[:, sg[seg]][:, None] * seg_sum
    return y


def reconstruct_f64(codes, books, scales, v: int, g: int) -> np.ndarray:
    """Decoded weights widened to binary64, for the tolerance oracle.

    Restates reconstruct (quantizer.py:428-452): centroid components summed
    in binary32 in codebook order, times the group scale in binary32, then
    rounded to f16.  The tolerance tests multiply this by x in binary64
    (test_acceptance.py:116, test_engines.py:273-281).
    """
    m = len(codes)
    rows, segs = codes[0].shape
    cols = segs * v
    w = np.zeros((rows, segs, v), dtype=np.float32)
    for t in range(m):
        w += np.asarray(books[t]).astype(np.float32)[codes[t]]
    sg = segment_groups(cols, v, g)
    w *= np.asarray(scales).astype(np.float32)[:, sg, None]
    return w.reshape(rows, cols).astype(F16).astype(np.float64)


# --------------------------------------------------------------------------
# code bit packing (quantizer.py:471-497)
# --------------------------------------------------------------------------

def pack_codes(codes: np.ndarray, b: int) -> bytes:
    """LSB-first b-bit stream, byte padded: code i owns bits [i*b, (i+1)*b)."""
    flat = np.asarray(codes, dtype=np.uint32).reshape(-1)
    bits = ((flat[:, None] >> np.arange(b, dtype=np.uint32)) & 1).astype(np.uint8)
    return np.packbits(bits.reshape(-1), bitorder="little").tobytes()


def unpack_codes(data: bytes, rows: int, segments: int, b: int) -> np.ndarray:
    count = rows * segments
    need = (count * b + 7) // 8
    bits = np.unpackbits(np.frombuffer(data, dtype=np.uint8, count=need), bitorder="little")
    bits = bits[: count * b].reshape(count, b).astype(np.uint32)
    vals = (bits << np.arange(b, dtype=np.uint32)).sum(axis=1, dtype=np.uint32)
    return vals.astype(np.uint16).reshape(rows, segments)


# --------------------------------------------------------------------------
# counters (accounting.py:109-126, engines.py:300-316)
# --------------------------------------------------------------------------

def closed_form_counters(rows: int, cols: int, n: int, v: int, m: int, b: int, t_w: int = 32):
    """The event tallies codegemm_gemm reports; bench.py:263-276 asserts them."""
    width = min(t_w, cols)
    events = m * rows * (cols // v) * n
    return {
        "mac_build": m * (1 << b) * cols * n,
        "mac_read_adds": events,
        "lookups": events,
        "mac_dense": 0,
        "psum_entries_per_tile": m * (1 << b) * (width // v),
    }


def rel_l2(y, ref) -> float:
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
