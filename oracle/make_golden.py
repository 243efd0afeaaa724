"""Generate tests/golden/*.npz from the REFERENCE package itself.

Run in the authoring container only (it imports /root/reference, which does
not exist on the GPU box):

    python oracle/make_golden.py

Every array written here is produced by calling the reference's own public
functions (engines.py, quantizer.py, bench.py); the committed fixtures are
what pins the oracle restatement (oracle/codegemm_oracle.py, cg_oracle.c)
and, through it, the CUDA path.  Test infrastructure only.
"""

from __future__ import annotations

import hashlib
import itertools
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def layer_digest(layer) -> str:
    return _digest([layer.scales.scales] + [b.entries for b in layer.books] + [p.codes for p in layer.planes])


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import codegemm as cg
    from codegemm import engines
    from codegemm.bench import ShapeSpec, bench_input, bench_layer

    os.makedirs(OUT, exist_ok=True)

    # ---- 1. psumbook known-answer tests (pkg/tests/test_engines.py:86-108)
    kat = {}
    book = cg.Codebook(np.array([[0, 1, 0, 0]], dtype=np.float16).repeat(2, axis=0))
    x = np.array([4.0, 7.0, -1.0, 2.5], dtype=np.float16)
    kat["unit_book"], kat["unit_x"] = book.entries, x
    kat["unit_out"] = cg.build_psumbook(x, [book]).entries
    book = cg.Codebook(np.ones((4, 2), dtype=np.float16))
    x = np.zeros(8, dtype=np.float16)
    kat["zero_book"], kat["zero_x"] = book.entries, x
    kat["zero_out"] = cg.build_psumbook(x, [book]).entries
    book = cg.Codebook(np.array([[1, 0], [0, 1], [1, 1], [-1, -1]], dtype=np.float16))
    x = np.array([2.0, 3.0], dtype=np.float16)
    ctr = cg.OpCounters()
    kat["dots_book"], kat["dots_x"] = book.entries, x
    kat["dots_out"] = cg.build_psumbook(x, [book], ctr).entries
    kat["dots_mac_build"] = np.int64(ctr.mac_build)
    # pack_codes KATs (pkg/tests/test_quantizer.py:243-250)
    kat["pack_b1_in"] = np.array([[1, 0, 1, 1]], dtype=np.uint16)
    kat["pack_b1_out"] = np.frombuffer(cg.pack_codes(cg.CodePlane(kat["pack_b1_in"]), 1), np.uint8)
    rng = np.random.default_rng(88)
    for b in (1, 2, 3, 4, 6, 8, 11, 16):
        codes = rng.integers(0, 2**b, size=(5, 11), dtype=np.uint16)
        kat[f"pack_b{b}_codes"] = codes
        kat[f"pack_b{b}_bytes"] = np.frombuffer(cg.pack_codes(cg.CodePlane(codes), b), np.uint8)
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **kat)

    # ---- 2. small layers: random_layer arrays, psum tables, engine outputs
    small = {}
    cases = [
        # (name, rows, cols, v, m, b, g, n, seed, t_w, t_h)
        ("grid_v2m1b2", 33, 32, 2, 1, 2, -1, 5, 2, 32, 2048),        # test_engines.py:168-179 grid
        ("grid_v4m2b4", 33, 64, 4, 2, 4, 8, 5, 4, 32, 2048),
        ("grid_v8m3b2", 33, 256, 8, 3, 2, 32, 5, 8, 32, 2048),
        ("grid_v16m1b8", 33, 128, 16, 1, 8, 16, 5, 16, 32, 2048),
        ("m1v4b8g128", 64, 512, 4, 1, 8, 128, 1, 11, 32, 2048),
        ("m2v8b8g128", 64, 512, 8, 2, 8, 128, 1, 12, 32, 2048),
        ("m1v4b8g128_n4", 48, 256, 4, 1, 8, 128, 4, 13, 32, 2048),
        ("partial_tile", 10, 80, 4, 1, 3, -1, 2, 9, 64, 8),           # test_engines.py:232-238
        ("th_threads", 40, 96, 4, 2, 4, 16, 3, 4, 32, 7),             # test_engines.py:220-229
        ("m1v8b8g128", 40, 1024, 8, 1, 8, 128, 1, 14, 32, 2048),
        ("m2v4b8g128", 40, 512, 4, 2, 8, 128, 1, 15, 32, 2048),
        ("m3v8b8g128", 24, 1024, 8, 3, 8, 128, 2, 16, 32, 2048),
        ("m4v8b8g128", 24, 1024, 8, 4, 8, 128, 1, 17, 32, 2048),
        ("m1v2b4g128", 40, 512, 2, 1, 4, 128, 1, 18, 32, 2048),
        ("m2v4b4g128", 40, 512, 4, 2, 4, 128, 1, 19, 32, 2048),
        ("m1v4b6g128", 40, 512, 4, 1, 6, 128, 1, 20, 32, 2048),
        ("m1v4b12g64", 16, 128, 4, 1, 12, 64, 2, 21, 32, 2048),
        ("g_row_ragged", 37, 200, 4, 1, 8, -1, 3, 22, 32, 2048),
    ]
    names = []
    for (name, rows, cols, v, m, b, g, n, seed, t_w, t_h) in cases:
        cfg = cg.QuantConfig(v=v, m=m, b=b, g=g, seed=seed)
        layer = cg.random_layer(rows, cols, cfg, seed=seed)
        xm = cg.Matrix.from_array(np.random.default_rng(seed + 1000).standard_normal((cols, n)))
        y, ctr = cg.codegemm_gemm(layer, xm, cg.TileConfig(t_w, t_h))
        ym, _ = cg.dequant_gemm(layer, xm, "mirrored")
        assert np.array_equal(y.view(np.uint32), ym.view(np.uint32))
        tables = engines._psum_tables([bk.widened() for bk in layer.books], xm.widened(), v)
        y64 = cg.reconstruct(layer).widened(np.float64) @ xm.widened(np.float64)
        p = name + "/"
        small[p + "meta"] = np.array([rows, cols, v, m, b, g, n, seed, t_w, t_h], dtype=np.int64)
        small[p + "scales"] = layer.scales.scales
        for t in range(m):
            small[p + f"book{t}"] = layer.books[t].entries
            small[p + f"codes{t}"] = layer.planes[t].codes
        small[p + "x"] = xm.data
        small[p + "y"] = y
        small[p + "y64"] = y64
        small[p + "tables"] = tables
        small[p + "counters"] = np.array(
            [ctr.mac_build, ctr.mac_read_adds, ctr.lookups, ctr.mac_dense, ctr.psum_entries_per_tile],
            dtype=np.int64,
        )
        small[p + "reconstruct"] = cg.reconstruct(layer).data
        names.append(name)
    small["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "small_layers.npz"), **small)

    # ---- 3. quantized (k-means) layers drawn like the acceptance sweep
    #      (test_acceptance.py:60-130): realistic codebooks, 24 cases.
    sweep = {}
    rng = np.random.default_rng(20260808)
    specs = list(itertools.product((2, 4, 8, 16), (1, 2, 3), (2, 4, 8)))
    picks = [specs[i] for i in rng.choice(len(specs), size=24, replace=False)]
    snames = []
    for i, (v, m, b) in enumerate(picks):
        g = [-1, v, 2 * v, 32][i % 4]
        base = v if g == -1 else g
        cols = base * int(rng.integers(1, max(1, 256 // base) + 1))
        rows = int(rng.integers(1, 97))
        n = int(rng.integers(1, 9))
        cfg = cg.QuantConfig(v=v, m=m, b=b, g=g, seed=int(rng.integers(2**32)), kmeans_iters=1)
        w = cg.Matrix.from_array(rng.standard_normal((rows, cols)))
        layer = cg.quantize_layer(w, cfg)
        xm = cg.Matrix.from_array(rng.standard_normal((cols, n)))
        y, _ = cg.codegemm_gemm(layer, xm)
        name = f"q{i:02d}"
        p = name + "/"
        sweep[p + "meta"] = np.array([rows, cols, v, m, b, g, n], dtype=np.int64)
        sweep[p + "scales"] = layer.scales.scales
        for t in range(m):
            sweep[p + f"book{t}"] = layer.books[t].entries
            sweep[p + f"codes{t}"] = layer.planes[t].codes
        sweep[p + "x"] = xm.data
        sweep[p + "y"] = y
        snames.append(name)
    sweep["names"] = np.array(snames)
    np.savez_compressed(os.path.join(OUT, "quantized_sweep.npz"), **sweep)

    # ---- 4. bench-shaped layers: generator digests + reference outputs
    big = {}
    shapes = [
        # (tag, B, N_out, K, v, m, b, g)
        ("8b_q_m1v4", 1, 4096, 4096, 4, 1, 8, 128),
        ("8b_q_m2v8", 1, 4096, 4096, 8, 2, 8, 128),
        ("8b_down_m1v4", 1, 4096, 14336, 4, 1, 8, 128),
        ("8b_q_m1v4_b4", 4, 4096, 4096, 4, 1, 8, 128),
    ]
    for tag, mb, n_out, k_in, v, m, b, g in shapes:
        cfg = cg.QuantConfig(v=v, m=m, b=b, g=g, seed=0)
        spec = ShapeSpec(m_batch=mb, n_out=n_out, k_in=k_in)
        layer = bench_layer(spec, cfg, 0)
        xm = bench_input(spec, 0)
        y, ctr = cg.codegemm_gemm(layer, xm, cg.TileConfig(32, 2048))
        p = tag + "/"
        big[p + "meta"] = np.array([mb, n_out, k_in, v, m, b, g], dtype=np.int64)
        big[p + "layer_sha256"] = np.array(layer_digest(layer))
        big[p + "x"] = xm.data
        big[p + "y"] = y
        big[p + "counters"] = np.array([ctr.mac_build, ctr.mac_read_adds], dtype=np.int64)
        print(tag, "done", flush=True)
    # criterion 3's large decode case (test_acceptance.py:186-192)
    cfg = cg.QuantConfig(v=4, m=1, b=8, g=128, seed=0)
    layer = cg.random_layer(4096, 14336, cfg, seed=1)
    xm = cg.Matrix.from_array(np.random.default_rng(2).standard_normal((14336, 1)))
    y, _ = cg.codegemm_gemm(layer, xm)
    big["crit3/layer_sha256"] = np.array(layer_digest(layer))
    big["crit3/x"] = xm.data
    big["crit3/y"] = y
    big["crit3/y64"] = cg.reconstruct(layer).widened(np.float64) @ xm.widened(np.float64)
    np.savez_compressed(os.path.join(OUT, "bench_shapes.npz"), **big)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
