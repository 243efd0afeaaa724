"""Pin the CPU oracle (numpy + C restatements) to the reference's own outputs.

Golden vectors in tests/golden were produced by the reference package itself
(oracle/make_golden.py); these tests prove the oracle reproduces them bit for
bit before any CUDA result is compared against the oracle.
"""

import hashlib

import numpy as np
import pytest

from oracle import c_oracle
from oracle import codegemm_oracle as orc


def u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def test_psumbook_kats_match_reference(kat):
    # pkg/tests/test_engines.py:86-108
    for tag in ("unit", "zero", "dots"):
        book = kat[f"{tag}_book"]
        x = kat[f"{tag}_x"]
        v = book.shape[1]
        got = orc.psum_tables([book.astype(np.float32)], x.astype(np.float32)[:, None], v)[..., 0]
        assert np.array_equal(u32(got), u32(kat[f"{tag}_out"])), tag
        got_c = c_oracle.psum_tables([book], x[:, None], v)[..., 0]
        assert np.array_equal(u32(got_c), u32(kat[f"{tag}_out"])), tag
    assert kat["unit_out"][0, 0, 0] == 7.0
    assert kat["dots_out"][0, 0].tolist() == [2.0, 3.0, 5.0, -5.0]
    assert int(kat["dots_mac_build"]) == 8


def test_pack_codes_kats(kat):
    # pkg/tests/test_quantizer.py:243-250: b=1 [1,0,1,1] -> 0b00001101
    assert orc.pack_codes(kat["pack_b1_in"], 1) == bytes(kat["pack_b1_out"])
    assert kat["pack_b1_out"].tolist() == [0b00001101]
    for b in (1, 2, 3, 4, 6, 8, 11, 16):
        codes = kat[f"pack_b{b}_codes"]
        packed = orc.pack_codes(codes, b)
        assert packed == bytes(kat[f"pack_b{b}_bytes"]), b
        assert np.array_equal(orc.unpack_codes(packed, *codes.shape, b), codes), b


def test_small_layers_tables_bit_exact(small_cases):
    for c in small_cases:
        books32 = [b.astype(np.float32) for b in c["books"]]
        got = orc.psum_tables(books32, c["x"].astype(np.float32), c["v"])
        assert np.array_equal(u32(got), u32(c["tables"])), c["name"]
        got_c = c_oracle.psum_tables(c["books"], c["x"], c["v"])
        assert np.array_equal(u32(got_c), u32(c["tables"])), c["name"]


def test_small_layers_engine_bit_exact(small_cases):
    for c in small_cases:
        t_w, t_h = int(c["meta"][8]), int(c["meta"][9])
        y = orc.codegemm(c["codes"], c["books"], c["scales"], c["x"], c["v"], c["g"], t_w, t_h)
        assert np.array_equal(u32(y), u32(c["y"])), c["name"]
        ym = orc.dequant_mirrored(c["codes"], c["books"], c["scales"], c["x"], c["v"], c["g"])
        assert np.array_equal(u32(ym), u32(c["y"])), c["name"]
        for threads in (1, 3):
            yc = c_oracle.codegemm(c["codes"], c["books"], c["scales"], c["x"], c["v"], c["g"],
                                   t_w, threads)
            assert np.array_equal(u32(yc), u32(c["y"])), (c["name"], threads)


def test_small_layers_reconstruct_and_counters(small_cases):
    for c in small_cases:
        w = orc.reconstruct_f64(c["codes"], c["books"], c["scales"], c["v"], c["g"])
        assert np.array_equal(w.astype(np.float16).view(np.uint16),
                              c["reconstruct"].view(np.uint16)), c["name"]
        t_w = int(c["meta"][8])
        cf = orc.closed_form_counters(c["rows"], c["cols"], c["n"], c["v"], c["m"], c["b"], t_w)
        assert [cf["mac_build"], cf["mac_read_adds"], cf["lookups"], cf["mac_dense"],
                cf["psum_entries_per_tile"]] == c["counters"].tolist(), c["name"]


def test_quantized_sweep_bit_exact(sweep_cases):
    for c in sweep_cases:
        y = orc.codegemm(c["codes"], c["books"], c["scales"], c["x"], c["v"], c["g"])
        assert np.array_equal(u32(y), u32(c["y"])), c["name"]
        yc = c_oracle.codegemm(c["codes"], c["books"], c["scales"], c["x"], c["v"], c["g"])
        assert np.array_equal(u32(yc), u32(c["y"])), c["name"]


def _digest(arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("tag", ["8b_q_m1v4", "8b_q_m2v8", "8b_q_m1v4_b4"])
def test_bench_shapes_generator_and_engine(bench_golden, tag):
    mb, n_out, k_in, v, m, b, g = (int(x) for x in bench_golden[f"{tag}/meta"])
    scales, books, codes = orc.random_layer_arrays(n_out, k_in, v, m, b, g,
                                                   orc.bench_layer_seed(n_out, k_in, 0))
    assert _digest([scales] + books + codes) == str(bench_golden[f"{tag}/layer_sha256"])
    x = orc.bench_input_array(k_in, mb, 0)
    assert np.array_equal(x.view(np.uint16), bench_golden[f"{tag}/x"].view(np.uint16))
    y = c_oracle.codegemm(codes, books, scales, x, v, g, threads=8)
    assert np.array_equal(u32(y), u32(bench_golden[f"{tag}/y"]))


def test_package_random_layer_matches_reference(bench_golden):
    import paper_2512_17970_b200 as cg

    for tag in ("8b_q_m1v4", "8b_q_m2v8"):
        mb, n_out, k_in, v, m, b, g = (int(x) for x in bench_golden[f"{tag}/meta"])
        q = cg.random_layer(n_out, k_in, cg.QuantConfig(v=v, m=m, b=b, g=g),
                            seed=orc.bench_layer_seed(n_out, k_in, 0))
        digest = _digest([q.scales.scales] + [bk.entries for bk in q.books]
                         + [p.codes for p in q.planes])
        assert digest == str(bench_golden[f"{tag}/layer_sha256"])
