"""GPU parity: the sm_100a kernels through the C ABI vs the pinned oracle.

Bit-exact: Psumbook contents (standalone K1 and the fused kernel's on-chip
table), per-row gather indices (unpacked prepack), strict-mode outputs.
Tolerance (fp32 accumulate, different order): fast-mode outputs, with the
tolerance written in helpers.py (norm. max-abs <= 1e-3, rel-L2 <= 1e-3,
per-element rel <= 1e-2 where |y| >= 1e-2 max|y|).
"""

import numpy as np
import pytest

import paper_2512_17970_b200 as cg
from paper_2512_17970_b200 import _lib
from helpers import assert_within_tolerance, layer_from_case, tolerance_report
from oracle import c_oracle
from oracle import codegemm_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def cuda_x(x16):
    return torch.from_numpy(np.ascontiguousarray(x16, dtype=np.float16)).cuda()


# ---------------------------------------------------------------- Psumbook


def test_psumbook_kats(kat):
    for tag in ("unit", "zero", "dots"):
        book = cg.Codebook(kat[f"{tag}_book"].copy())
        ctr = cg.OpCounters()
        got = cg.build_psumbook(kat[f"{tag}_x"], [book], ctr)
        assert np.array_equal(u32(got.entries), u32(kat[f"{tag}_out"])), tag
    got = cg.build_psumbook(kat["dots_x"], [cg.Codebook(kat["dots_book"].copy())], ctr := cg.OpCounters())
    assert got.entries[0, 0].tolist() == [2.0, 3.0, 5.0, -5.0] and ctr.mac_build == 8
    zero = cg.build_psumbook(kat["zero_x"], [cg.Codebook(kat["zero_book"].copy())])
    assert not zero.entries.any() and zero.entry_count == 16


def test_standalone_psumbook_bit_exact(small_cases):
    from paper_2512_17970_b200 import _lib
    import ctypes

    lib = _lib.load()
    for c in small_cases:
        books = torch.from_numpy(np.concatenate([b.reshape(-1) for b in c["books"]])).cuda()
        x = cuda_x(c["x"])
        k = 1 << c["b"]
        out = torch.empty((c["m"], c["cols"] // c["v"], k, c["n"]), dtype=torch.float32,
                          device="cuda")
        _lib.check(lib.cg_psumbook_build(books.data_ptr(), x.data_ptr(), c["m"], c["b"], c["v"],
                                         c["cols"], c["n"], out.data_ptr(), None))
        torch.cuda.synchronize()
        assert np.array_equal(u32(out.cpu().numpy()), u32(c["tables"])), c["name"]


def test_fused_kernel_psumbook_bit_exact(small_cases):
    seen = 0
    for c in small_cases:
        dl = cg.DeviceLayer(layer_from_case(c))
        if not dl.info["fast_supported"]:
            continue
        got = dl.psumbook(cuda_x(c["x"]))
        torch.cuda.synchronize()
        assert np.array_equal(u32(got.cpu().numpy()), u32(c["tables"])), c["name"]
        seen += 1
    assert seen >= 10


def test_fused_psumbook_all_tilings():
    q = cg.random_layer(40, 1024, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=5)
    x = orc.bench_input_array(1024, 3, 7)
    ref = orc.psum_tables([b.entries.astype(np.float32) for b in q.books], x.astype(np.float32), 4)
    for u in (1, 2, 4):
        got = cg.DeviceLayer(q, u=u).psumbook(cuda_x(x)).cpu().numpy()
        assert np.array_equal(u32(got), u32(ref)), u


# ---------------------------------------------------------------- gather indices


def test_unpacked_codes_equal_reference_planes(small_cases, sweep_cases):
    for c in small_cases + sweep_cases:
        dl = cg.DeviceLayer(layer_from_case(c))
        got = dl.unpack_codes()
        want = np.stack(c["codes"])
        assert got.dtype == np.uint16 and np.array_equal(got, want), c["name"]


def test_unpacked_codes_all_tilings_ragged():
    q = cg.random_layer(37, 4 * 200, cg.QuantConfig(v=4, m=2, b=8, g=-1), seed=3)
    want = np.stack([p.codes for p in q.planes])
    for u in (1, 2):
        assert np.array_equal(cg.DeviceLayer(q, u=u).unpack_codes(), want), u


# ---------------------------------------------------------------- outputs


def test_strict_mode_bit_exact(small_cases, sweep_cases):
    for c in small_cases + sweep_cases:
        q = layer_from_case(c)
        y, ctr = cg.codegemm_gemm(q, cg.Matrix(c["x"]), mode="strict")
        assert np.array_equal(u32(y), u32(c["y"])), c["name"]


def test_fast_mode_within_tolerance(small_cases, sweep_cases):
    fast = 0
    for c in small_cases + sweep_cases:
        q = layer_from_case(c)
        y, ctr = cg.codegemm_gemm(q, cg.Matrix(c["x"]), mode="auto")
        assert_within_tolerance(y, c["y"], c["name"])
        fast += cg.DeviceLayer(q).info["fast_supported"]
    assert fast >= 20


def test_fast_mode_counters_match_reference(small_cases):
    for c in small_cases:
        t_w, t_h = int(c["meta"][8]), int(c["meta"][9])
        _, ctr = cg.codegemm_gemm(layer_from_case(c), cg.Matrix(c["x"]), cg.TileConfig(t_w, t_h))
        assert [ctr.mac_build, ctr.mac_read_adds, ctr.lookups, ctr.mac_dense,
                ctr.psum_entries_per_tile] == c["counters"].tolist(), c["name"]


def test_zero_input_gives_zero_and_counts():
    # pkg/tests/test_engines.py:160-165
    layer = cg.random_layer(8, 32, cg.QuantConfig(v=4, m=2, b=3, g=8, seed=1), seed=2)
    y, counters = cg.codegemm_gemm(layer, cg.Matrix.from_array(np.zeros((32, 3))))
    assert not y.any()
    assert counters.lookups == 2 * 8 * (32 // 4) * 3


@pytest.mark.parametrize("tag", ["8b_q_m1v4", "8b_q_m2v8", "8b_q_m1v4_b4"])
def test_bench_shapes_vs_reference(bench_golden, tag):
    mb, n_out, k_in, v, m, b, g = (int(x) for x in bench_golden[f"{tag}/meta"])
    q = cg.random_layer(n_out, k_in, cg.QuantConfig(v=v, m=m, b=b, g=g),
                        seed=orc.bench_layer_seed(n_out, k_in, 0))
    x = cg.Matrix(bench_golden[f"{tag}/x"])
    y, _ = cg.codegemm_gemm(q, x)
    assert_within_tolerance(y, bench_golden[f"{tag}/y"], tag)
    ys, _ = cg.codegemm_gemm(q, x, mode="strict")
    assert np.array_equal(u32(ys), u32(bench_golden[f"{tag}/y"])), tag


def test_criterion3_large_decode_shape(bench_golden):
    # test_acceptance.py:186-192: (1, 4096, 14336) m1v4b8g128 rel-L2 <= 1e-3 vs binary64
    q = cg.random_layer(4096, 14336, cg.QuantConfig(v=4, m=1, b=8, g=128, seed=0), seed=1)
    y, _ = cg.codegemm_gemm(q, cg.Matrix(bench_golden["crit3/x"]))
    assert orc.rel_l2(y, bench_golden["crit3/y64"]) <= 1e-3
    assert_within_tolerance(y, bench_golden["crit3/y"], "crit3")


def test_longest_reduction_tolerance():
    # test_engines.py:273-281: K=32768 rel-L2 <= 1e-3 vs binary64
    q = cg.random_layer(8, 32768, cg.QuantConfig(v=4, m=1, b=8, g=128, seed=0), seed=1)
    x = np.random.default_rng(2).standard_normal((32768, 2)).astype(np.float16)
    y, _ = cg.codegemm_gemm(q, cg.Matrix(x))
    codes = [p.codes for p in q.planes]
    books = [b.entries for b in q.books]
    w = orc.reconstruct_f64(codes, books, q.scales.scales, 4, 128)
    assert orc.rel_l2(y, w @ x.astype(np.float64)) <= 1e-3


@pytest.mark.parametrize("shape", [(28672, 8192), (8192, 28672), (14336, 4096)])
def test_full_size_70b_shapes_vs_c_oracle(shape):
    rows, cols = shape
    for v, m in ((4, 1), (8, 2)):
        q = cg.random_layer(rows, cols, cg.QuantConfig(v=v, m=m, b=8, g=128),
                            seed=orc.bench_layer_seed(rows, cols, 0))
        x = orc.bench_input_array(cols, 1, 0)
        y, _ = cg.codegemm_gemm(q, cg.Matrix(x))
        ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                                q.scales.scales, x, v, 128, threads=8)
        assert_within_tolerance(y, ref, f"{shape} m{m}v{v}")


# ---------------------------------------------------------------- invariances


DET = _lib.CG_OPT_DETERMINISTIC


def test_fast_mode_deterministic_and_tiling_invariant_per_u():
    # deterministic split-K: bits independent of run, rows per task, grid waves
    q = cg.random_layer(1000, 4096, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=11)
    x = cuda_x(orc.bench_input_array(4096, 1, 3))
    for u in (1, 2, 4):
        ref = cg.DeviceLayer(q, u=u, flags=DET).gemm(x).cpu().numpy()
        again = cg.DeviceLayer(q, u=u, flags=DET).gemm(x).cpu().numpy()
        assert np.array_equal(u32(ref), u32(again))
        for rg in (1, 3, 16, 63):
            y = cg.DeviceLayer(q, u=u, rg_per_task=rg, flags=DET).gemm(x).cpu().numpy()
            assert np.array_equal(u32(y), u32(ref)), (u, rg)
            # default split-K (L2 reduce-add): same values up to fp32 add order
            y2 = cg.DeviceLayer(q, u=u, rg_per_task=rg).gemm(x).cpu().numpy()
            assert_within_tolerance(y2, ref, f"reduce-add u={u} rg={rg}")


def test_row_shards_bit_identical_to_full_layer():
    q = cg.random_layer(1000, 2048, cg.QuantConfig(v=8, m=2, b=8, g=128), seed=12)
    x = cuda_x(orc.bench_input_array(2048, 1, 4))
    full = cg.DeviceLayer(q, u=2, flags=DET).gemm(x).cpu().numpy()
    bounds = [0, 250, 500, 750, 1000]
    parts = [cg.DeviceLayer(q, u=2, row_range=(a, b), flags=DET).gemm(x).cpu().numpy()
             for a, b in zip(bounds, bounds[1:])]
    assert np.array_equal(u32(np.concatenate(parts)), u32(full))


def test_strict_independent_of_tiling():
    q = cg.random_layer(40, 96, cg.QuantConfig(v=4, m=2, b=4, g=16, seed=3), seed=4)
    x = np.random.default_rng(5).standard_normal((96, 3)).astype(np.float16)
    ref = orc.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                       q.scales.scales, x, 4, 16)
    for u in (1, 2):
        y = cg.DeviceLayer(q, u=u).gemm(cuda_x(x), mode="strict").cpu().numpy()
        assert np.array_equal(u32(y), u32(ref)), u


def test_host_and_device_entry_points_agree():
    q = cg.random_layer(300, 1024, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=9)
    x = orc.bench_input_array(1024, 2, 9)
    dl = cg.DeviceLayer(q, flags=DET)
    y_host = dl.gemm_host(x)
    y_dev = dl.gemm(cuda_x(x)).cpu().numpy()
    assert np.array_equal(u32(y_host), u32(y_dev))


def test_integrity_error_for_out_of_range_code():
    from types import SimpleNamespace

    codes = np.zeros((4, 8), np.uint16)
    codes[1, 3] = 300
    fake = SimpleNamespace(
        rows=4, cols=32, config=SimpleNamespace(v=4, m=1, b=8, g=-1),
        planes=(SimpleNamespace(codes=codes),),
        books=(SimpleNamespace(entries=np.zeros((256, 4), np.float16)),),
        scales=SimpleNamespace(scales=np.ones((4, 1), np.float16)),
    )
    with pytest.raises(cg.IntegrityError):
        cg.DeviceLayer(fake)


def test_fast_mode_rejected_when_unsupported():
    q = cg.random_layer(16, 128, cg.QuantConfig(v=4, m=1, b=12, g=64), seed=1)
    dl = cg.DeviceLayer(q)
    assert not dl.info["fast_supported"]
    with pytest.raises(cg.ConfigError):
        dl.gemm_host(np.ones((128, 1), np.float16), mode="fast")


def test_group_launch_bit_identical_to_single_launches():
    shapes = [(300, 1024), (4096, 512), (37, 2048), (1000, 4096), (64, 128)]
    layers, xs, refs = [], [], []
    for i, (r, c) in enumerate(shapes):
        q = cg.random_layer(r, c, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=40 + i)
        dl = cg.DeviceLayer(q, flags=DET)
        x = cuda_x(orc.bench_input_array(c, 2, i))
        layers.append(dl)
        xs.append(x)
        refs.append(dl.gemm(x).cpu().numpy())
    ys = cg.gemm_group(layers, xs)
    for y, ref in zip(ys, refs):
        assert np.array_equal(u32(y.cpu().numpy()), u32(ref))
    # and again (tickets are monotonic across calls)
    ys = cg.gemm_group(layers, xs)
    for y, ref in zip(ys, refs):
        assert np.array_equal(u32(y.cpu().numpy()), u32(ref))


def test_repeated_calls_stable():
    q = cg.random_layer(2000, 8192, cg.QuantConfig(v=8, m=2, b=8, g=128), seed=77)
    dl = cg.DeviceLayer(q, flags=DET)
    x = cuda_x(orc.bench_input_array(8192, 1, 5))
    ref = dl.gemm(x).cpu().numpy()
    for _ in range(5):
        assert np.array_equal(u32(dl.gemm(x).cpu().numpy()), u32(ref))


def test_group_launch_default_mode_within_tolerance():
    layers, xs, refs = [], [], []
    for i, (r, c) in enumerate([(4096, 4096), (14336, 4096), (4096, 14336)]):
        q = cg.random_layer(r, c, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=90 + i)
        x16 = orc.bench_input_array(c, 1, i)
        layers.append(cg.DeviceLayer(q))
        xs.append(cuda_x(x16))
        refs.append(c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                                      q.scales.scales, x16, 4, 128, threads=8))
    for _ in range(3):
        ys = cg.gemm_group(layers, xs)
        for y, ref in zip(ys, refs):
            assert_within_tolerance(y.cpu().numpy(), ref, "group reduce-add")


# ---------------------------------------------------------------- staged launches
def _chain(shapes, cfg, seed, u, flags=0):
    layers = [cg.DeviceLayer(cg.random_layer(r, c, cfg, seed=seed + i), u=u, flags=flags)
              for i, (r, c) in enumerate(shapes)]
    return layers


@pytest.mark.parametrize("det", [True, False])
def test_staged_chain_matches_separate_launches(det):
    """x of stage s+1 is y of stage s (float32, rounded to binary16 as read):
    the in-kernel grid barrier orders it; bit-identical to separate launches
    on the torch-rounded inputs in deterministic mode, within tolerance in
    reduce-add mode."""
    cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
    shapes = [(1024, 2048), (4096, 1024), (2048, 4096), (512, 2048)]
    layers = _chain(shapes, cfg, 300, u=2, flags=DET if det else 0)
    x0 = cuda_x(orc.bench_input_array(2048, 1, 3))
    ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, _ in shapes]
    xs = [x0] + ys[:-1]
    for _ in range(3):  # repeated launches: barrier counters carry over
        for y in ys:
            y.fill_(float("nan"))
        cg.gemm_stages(layers, xs, ys, [0, 1, 2, 3])
        ref_x = x0
        for dl, y in zip(layers, ys):
            ref = dl.gemm(ref_x)
            if det:
                assert np.array_equal(u32(y.cpu().numpy()), u32(ref.cpu().numpy()))
            else:
                assert_within_tolerance(y.cpu().numpy(), ref.cpu().numpy(), "staged chain")
            ref_x = y.half()  # the next stage's input, as the kernel rounded it


def test_staged_block_vs_c_oracle():
    """Decoder-block chain {q,k,v} -> {o} -> {gate,up} -> {down} in one launch
    (k/v GQA-shaped), every stage against the C oracle on the fp16-rounded
    output of the stage before."""
    cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
    H, F, KV = 1024, 3584, 256
    shapes = [(H, H), (KV, H), (KV, H), (H, H), (F, H), (F, H), (H, F)]
    stages = [0, 0, 0, 1, 2, 2, 3]
    qs = [cg.random_layer(r, c, cfg, seed=500 + i) for i, (r, c) in enumerate(shapes)]
    layers = [cg.DeviceLayer(q, u=2) for q in qs]
    x0 = orc.bench_input_array(H, 1, 9)
    ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, _ in shapes]
    src = {0: None, 1: None, 2: None, 3: 0, 4: 3, 5: 3, 6: 4}  # x source (layer index)
    xs = [cuda_x(x0) if src[i] is None else ys[src[i]] for i in range(7)]
    cg.gemm_stages(layers, xs, ys, stages)
    got = [y.cpu().numpy() for y in ys]
    for i, q in enumerate(qs):
        xin = x0 if src[i] is None else got[src[i]].astype(np.float16)
        ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                                q.scales.scales, xin, 4, 128, threads=8)
        assert_within_tolerance(got[i], ref, f"block stage layer {i}")


@pytest.mark.parametrize("contig", [True, False])
def test_independent_block_one_stage_vs_c_oracle(contig, monkeypatch):
    """The 8B block's 7 layers as independent layers in ONE stage: several tasks
    per CTA, so with contiguous task ranges (default) consecutive tasks of a CTA
    reuse the Psumbook of their (layer, K-slice) without a rebuild.  Every layer
    against the C oracle; the strided schedule (CG_NO_CONTIG) gives the same
    rows up to the split-K reduce-add order."""
    if not contig:
        monkeypatch.setenv("CG_NO_CONTIG", "1")
    cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
    shapes = [(4096, 4096)] * 4 + [(14336, 4096)] * 2 + [(4096, 14336)]
    qs = [cg.random_layer(r, c, cfg, seed=900 + i) for i, (r, c) in enumerate(shapes)]
    layers = [cg.DeviceLayer(q, u=4) for q in qs]
    xs16 = [orc.bench_input_array(c, 1, 40 + i) for i, (r, c) in enumerate(shapes)]
    ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, _ in shapes]
    plan = cg.StagedLaunch(layers, [cuda_x(x) for x in xs16], ys, [0] * len(shapes))
    plan()
    got = [y.cpu().numpy() for y in ys]
    for i, q in enumerate(qs):
        ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                                q.scales.scales, xs16[i], 4, 128, threads=8)
        assert_within_tolerance(got[i], ref, f"independent layer {i} (contig={contig})")
        assert orc.rel_l2(got[i], ref) <= 1e-5
    plan()  # a second launch of the prepared plan: same rows
    for i in range(len(shapes)):
        assert orc.rel_l2(ys[i].cpu().numpy(), got[i]) <= 1e-6


def test_staged_launch_rejects_unaligned_output():
    q = cg.random_layer(256, 1024, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=31)
    dl = cg.DeviceLayer(q, u=2)
    x = cuda_x(orc.bench_input_array(1024, 1, 3))
    buf = torch.empty(256 + 1, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        cg.gemm_stages([dl], [x], [buf[1:].view(256, 1)], [0])


def test_staged_launch_rejects_mixed_tiling_and_bad_stages():
    cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
    a = cg.DeviceLayer(cg.random_layer(256, 1024, cfg, seed=1), u=2)
    b = cg.DeviceLayer(cg.random_layer(256, 1024, cfg, seed=2), u=4)
    x = cuda_x(orc.bench_input_array(1024, 1, 0))
    ys = [torch.empty((256, 1), dtype=torch.float32, device="cuda") for _ in range(2)]
    with pytest.raises(cg.ConfigError):
        cg.gemm_stages([a, b], [x, x], ys, [0, 1])
    with pytest.raises(ValueError):
        cg.gemm_stages([a, a], [x, x], ys, [0, 2])


@pytest.mark.parametrize("n", [4, 8])
def test_multi_column_direct_add_vs_c_oracle(n):
    """n > 1 in reduce-add mode adds split-K partials straight into y (red.add)."""
    q = cg.random_layer(3000, 4096, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=60 + n)
    x16 = orc.bench_input_array(4096, n, n)
    ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                            q.scales.scales, x16, 4, 128, threads=8)
    for u in (2, 4):
        dl = cg.DeviceLayer(q, u=u)
        for _ in range(2):
            assert_within_tolerance(dl.gemm(cuda_x(x16)).cpu().numpy(), ref, f"n={n} u={u}")


def test_staged_chain_m2v8():
    """The second 2-bit configuration (m2v8g128) through a dependent staged chain."""
    cfg = cg.QuantConfig(v=8, m=2, b=8, g=128)
    shapes = [(2048, 1024), (1024, 2048), (3072, 1024)]
    qs = [cg.random_layer(r, c, cfg, seed=700 + i) for i, (r, c) in enumerate(shapes)]
    layers = [cg.DeviceLayer(q, u=1) for q in qs]
    x0 = orc.bench_input_array(1024, 1, 4)
    ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, _ in shapes]
    cg.gemm_stages(layers, [cuda_x(x0), ys[0], ys[1]], ys, [0, 1, 2])
    got = [y.cpu().numpy() for y in ys]
    xin = x0
    for i, q in enumerate(qs):
        ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                                q.scales.scales, xin, 8, 128, threads=8)
        assert_within_tolerance(got[i], ref, f"m2v8 stage {i}")
        xin = got[i].astype(np.float16)


def test_prepared_staged_launch_and_host_entry():
    """StagedLaunch (cg_stages_prepare/launch/run_host): bit-identical to
    gemm_stages in deterministic mode, end to end with pinned host buffers, and
    re-planned when a wider call reallocated a layer's split-K workspace."""
    cfg = cg.QuantConfig(v=4, m=1, b=8, g=128)
    shapes = [(1024, 2048), (2048, 1024), (512, 2048)]
    layers = _chain(shapes, cfg, 900, u=2, flags=DET)
    x0 = cuda_x(orc.bench_input_array(2048, 1, 5))
    ref_ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, _ in shapes]
    cg.gemm_stages(layers, [x0] + ref_ys[:-1], ref_ys, [0, 1, 2])
    ref = [y.cpu().numpy() for y in ref_ys]
    ybuf = torch.empty(sum(r for r, _ in shapes), dtype=torch.float32, device="cuda")
    offs = np.cumsum([0] + [r for r, _ in shapes])
    ys = [ybuf[a:b].view(-1, 1) for a, b in zip(offs, offs[1:])]
    xdev = torch.empty_like(x0)
    plan = cg.StagedLaunch(layers, [xdev] + ys[:-1], ys, [0, 1, 2])
    xdev.copy_(x0)
    for _ in range(2):
        ybuf.fill_(float("nan"))
        plan()
        for y, r in zip(ys, ref):
            assert np.array_equal(u32(y.cpu().numpy()), u32(r))
    host_x = x0.cpu().pin_memory()
    host_y = torch.empty(ybuf.numel(), dtype=torch.float32).pin_memory()
    xdev.zero_()
    plan.run_host(host_x, xdev, ybuf, host_y)
    assert np.array_equal(u32(host_y.numpy()), u32(np.concatenate(ref).reshape(-1)))
    host_y.fill_(float("nan"))
    step = plan.bind_host(host_x, xdev, ybuf, host_y)
    step()
    assert np.array_equal(u32(host_y.numpy()), u32(np.concatenate(ref).reshape(-1)))
    # a wider call on the first layer reallocates its workspace: the plan re-plans
    layers[0].gemm(cuda_x(orc.bench_input_array(2048, 4, 6)))
    ybuf.fill_(float("nan"))
    plan()
    for y, r in zip(ys, ref):
        assert np.array_equal(u32(y.cpu().numpy()), u32(r))
