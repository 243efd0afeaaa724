"""Host-side behaviour of the drop-in API (no GPU needed).

Mirrors the reference's own argument-checking tests
(pkg/tests/test_engines.py:30-46, 241-270) against this package.
"""

import numpy as np
import pytest

import paper_2512_17970_b200 as cg
from paper_2512_17970_b200.engines import closed_form_counters


def test_tile_config_validation():
    with pytest.raises(cg.ConfigError):
        cg.TileConfig(0, 2048)
    with pytest.raises(cg.ConfigError):
        cg.TileConfig(32, 0)
    cfg = cg.QuantConfig(v=8, m=1, b=2, g=16)
    cg.TileConfig(32, 4).validate_for(cfg)
    with pytest.raises(cg.ConfigError):
        cg.TileConfig(12, 4).validate_for(cfg)
    with pytest.raises(cg.ConfigError):
        cg.TileConfig(t_w=4, t_h=4).validate_for(cg.QuantConfig(v=8, m=1, b=2))
    with pytest.raises(cg.ConfigError):
        cg.TileConfig(48, 4).validate_for(cg.QuantConfig(v=4, m=1, b=2, g=32))
    cg.TileConfig(64, 4).validate_for(cg.QuantConfig(v=4, m=1, b=2, g=32))
    cg.TileConfig(16, 4).validate_for(cg.QuantConfig(v=4, m=1, b=2, g=32))


def test_quant_config_rules():
    for kw in (dict(v=0, m=1, b=2), dict(v=2, m=0, b=2), dict(v=2, m=1, b=0),
               dict(v=2, m=1, b=17), dict(v=4, m=1, b=2, g=2), dict(v=4, m=1, b=2, g=6),
               dict(v=2, m=1, b=2, kmeans_iters=0)):
        with pytest.raises(cg.ConfigError):
            cg.QuantConfig(**kw)
    with pytest.raises(cg.ConfigError):
        cg.QuantConfig(v=4, m=1, b=2).validate_shape(3, 6)
    with pytest.raises(cg.ConfigError):
        cg.QuantConfig(v=4, m=1, b=2, g=8).validate_shape(3, 12)


def test_container_integrity():
    with pytest.raises(cg.IntegrityError):
        cg.Codebook(np.zeros((3, 2), np.float16))
    with pytest.raises(cg.IntegrityError):
        cg.Codebook(np.full((4, 2), np.inf, np.float16))
    with pytest.raises(cg.IntegrityError):
        cg.ScalePlane(np.zeros((2, 2), np.float16))
    with pytest.raises(cg.IntegrityError):
        cg.CodePlane(np.zeros((2, 2), np.int32))
    cfg = cg.QuantConfig(v=2, m=1, b=2)
    good = dict(rows=2, cols=4, config=cfg, scales=cg.ScalePlane(np.ones((2, 1), np.float16)),
                planes=(cg.CodePlane(np.zeros((2, 2), np.uint16)),),
                books=(cg.Codebook(np.zeros((4, 2), np.float16)),))
    cg.QuantizedLayer(**good)
    bad = dict(good, planes=(cg.CodePlane(np.full((2, 2), 4, np.uint16)),))
    with pytest.raises(cg.IntegrityError):
        cg.QuantizedLayer(**bad)
    with pytest.raises(cg.IntegrityError):
        cg.QuantizedLayer(**dict(good, books=()))


def test_codegemm_argument_errors_precede_device_use():
    # engines.py:264-269 order: shape, then tiling, then threads
    layer = cg.random_layer(8, 32, cg.QuantConfig(v=4, m=1, b=2), seed=0)
    with pytest.raises(cg.ShapeError):
        cg.codegemm_gemm(layer, cg.Matrix.from_array(np.zeros((16, 2))))
    x = cg.Matrix.from_array(np.zeros((32, 2)))
    with pytest.raises(cg.ConfigError):
        cg.codegemm_gemm(layer, x, cg.TileConfig(t_w=6, t_h=8))
    with pytest.raises(cg.ConfigError):
        cg.codegemm_gemm(layer, x, threads=0)
    with pytest.raises(cg.ConfigError):
        cg.codegemm_gemm(layer, x, mode="sideways")


def test_phase_split_and_counters():
    assert cg.phase_split(cg.OpCounters(mac_build=10, mac_read_adds=10)) == (0.5, 0.5)
    assert cg.phase_split(cg.OpCounters(mac_build=1, mac_read_adds=3)) == (0.25, 0.75)
    with pytest.raises(ValueError):
        cg.phase_split(cg.OpCounters())
    # pkg/tests/test_engines.py:209-217 at 4096x4096 m1v4b8
    c = closed_form_counters(4096, 4096, 1, 4, 1, 8, 32)
    assert c.mac_read_adds == 4_194_304 and c.mac_build == 1_048_576
    assert c.lookups == c.mac_read_adds
    # test_engines.py:241-248 space claim: m*2**b*t_w/v < m*2**b*v iff t_w < v**2
    c = closed_form_counters(8, 64, 1, 8, 2, 4, 32)
    assert c.psum_entries_per_tile == 2 * 2**4 * (32 // 8) < 2 * 2**4 * 8


def test_pack_unpack_round_trip():
    rng = np.random.default_rng(88)
    for b in range(1, 17):
        codes = rng.integers(0, 2**b, size=(5, 11), dtype=np.uint16)
        back = cg.unpack_codes(cg.pack_codes(cg.CodePlane(codes), b), 5, 11, b)
        assert np.array_equal(back.codes, codes)


def test_matrix_container():
    m = cg.Matrix.from_array([[1.5, -2.0], [np.nan, 8.0]])
    assert m.bits[1, 0] == 0x7E00
    assert not m.data.flags.writeable
    with pytest.raises(cg.ShapeError):
        cg.Matrix(np.zeros((2, 2), np.float32))


def test_gemm_stages_argument_checks():
    """gemm_stages validates shapes and dtypes before touching the library."""
    torch = pytest.importorskip("torch")

    class FakeLayer:  # the attributes gemm_stages reads before the launch
        def __init__(self, rows, cols):
            self.rows, self.cols = rows, cols

    a, b = FakeLayer(64, 128), FakeLayer(32, 64)
    x = torch.zeros((128, 1), dtype=torch.float16)
    ya = torch.zeros((64, 1), dtype=torch.float32)
    yb = torch.zeros((32, 1), dtype=torch.float32)
    with pytest.raises(cg.ShapeError):  # one x/y/stage per layer
        cg.gemm_stages([a, b], [x], [ya, yb], [0, 1])
    with pytest.raises(cg.ShapeError):  # x rows must be the layer's cols
        cg.gemm_stages([a, b], [x, x], [ya, yb], [0, 1])
    with pytest.raises(cg.ShapeError):  # x must be float16 or float32
        cg.gemm_stages([a], [x.to(torch.float64)], [ya], [0])
    with pytest.raises(cg.ShapeError):  # y must be (rows, n) float32
        cg.gemm_stages([a], [x], [ya.to(torch.float16)], [0])
    with pytest.raises(cg.ShapeError):
        cg.gemm_stages([a], [x], [yb], [0])
    # prepared launches check the same, plus the exchange arguments
    with pytest.raises(cg.ShapeError):
        cg.StagedLaunch([a, b], [x], [ya, yb], [0, 1])
    with pytest.raises(cg.ConfigError):  # exchange flags without a comm
        cg.StagedLaunch([a], [x], [ya], [0], xchg=[1])
    with pytest.raises(cg.ShapeError):  # one flag per layer
        cg.StagedLaunch([a], [x], [ya], [0], xchg=[1, 1], comm=object())
