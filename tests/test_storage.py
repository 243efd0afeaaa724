"""The CGMM container (storage.py of the reference) and the GPU loader.

CPU: files written by the reference's own serializer (oracle/make_cgmm_golden.py) decode to the
reference-decoded planes, scales and codebooks; the reference's error classes for bad magic,
version, truncation and trailing bytes; serialize/deserialize round trip.
GPU: load_device_layer unpacks the b-bit planes on the device -- the unpacked gather indices
equal the reference planes bit for bit and the outputs match the oracle.
"""

import os

import numpy as np
import pytest

import paper_2512_17970_b200 as cg
from helpers import assert_within_tolerance
from oracle import c_oracle
from oracle import codegemm_oracle as orc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["m1v4b8g128", "m2v8b8g128", "m1v4b3grow", "m2v4b6g64"]


@pytest.fixture(scope="module")
def planes():
    with np.load(os.path.join(GOLD, "cgmm_planes.npz")) as z:
        return {k: z[k] for k in z.files}


def path_of(name):
    return os.path.join(GOLD, "cgmm", name + ".cgmm")


@pytest.mark.parametrize("name", CASES)
def test_deserialize_matches_reference_decode(name, planes):
    q = cg.deserialize(path_of(name))
    for t in range(q.config.m):
        assert np.array_equal(q.planes[t].codes, planes[f"{name}/codes{t}"])
        assert np.array_equal(q.books[t].entries.view(np.uint16),
                              planes[f"{name}/book{t}"].view(np.uint16))
    assert np.array_equal(q.scales.scales.view(np.uint16), planes[f"{name}/scales"].view(np.uint16))


@pytest.mark.parametrize("name", CASES)
def test_serialize_round_trip_is_byte_identical(name, tmp_path):
    q = cg.deserialize(path_of(name))
    out = tmp_path / "again.cgmm"
    cg.serialize(q, out)
    assert open(out, "rb").read() == open(path_of(name), "rb").read()


def test_format_errors(tmp_path):
    raw = open(path_of("m1v4b8g128"), "rb").read()
    cases = [(b"XXXX" + raw[4:], cg.BadMagicError),
             (raw[:2], cg.TruncatedFileError),
             (raw[:30], cg.TruncatedFileError),
             (raw[:4] + (2).to_bytes(4, "little") + raw[8:], cg.UnsupportedVersionError),
             (raw[:-5], cg.TruncatedFileError),
             (raw + b"\0", cg.IntegrityError)]
    for i, (data, exc) in enumerate(cases):
        p = tmp_path / f"bad{i}.cgmm"
        p.write_bytes(data)
        with pytest.raises(exc):
            cg.deserialize(p)
        assert issubclass(exc, cg.CodeGemmError)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_loader_index_parity_and_outputs(name, planes):
    torch = pytest.importorskip("torch")
    dl = cg.load_device_layer(path_of(name))
    want = np.stack([planes[f"{name}/codes{t}"] for t in range(dl.m)])
    assert np.array_equal(dl.unpack_codes(), want)  # b-bit planes unpacked on the device
    q = cg.deserialize(path_of(name))
    x16 = orc.bench_input_array(q.cols, 2, 5)
    ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                            q.scales.scales, x16, q.config.v, q.config.g, threads=4)
    y = dl.gemm(torch.from_numpy(x16).cuda()).cpu().numpy()
    assert_within_tolerance(y, ref, name)
    ys = dl.gemm(torch.from_numpy(x16).cuda(), mode="strict").cpu().numpy()
    assert np.array_equal(ys.view(np.uint32), ref.view(np.uint32))
