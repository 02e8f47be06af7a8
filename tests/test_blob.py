"""State-blob + sidecar I/O (layout.hpp:155-200) through the C ABI
(hf_blob_info / hf_blob_read / hf_blob_write), pinned to the reference's own
export_blob / import_blob (oracle/_ref, compiled from /root/reference): blobs the
reference writes parse bit-exactly, blobs the library writes are byte-identical to
the reference's and read back by it, and the reference's error classes map to
HF_ERUNTIME / HF_EINVAL.  Host only (no GPU)."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2107_14027_b200 as hf
from paper_2107_14027_b200 import HexfuseError, HexfuseInvalid, Precision

ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (reference tree absent)")

SHAPES = [(3, 2, 6, 4, True), (3, 3, 45, 32, False), (2, 5, 13, 7, True), (3, 1, 1, 1, False), (2, 8, 9, 4, False)]


def _files(path):
    with open(path, "rb") as a, open(path + ".json", "rb") as b:
        return a.read(), b.read()


@ref_only
@pytest.mark.parametrize("d,p,n,g,fp32", SHAPES)
def test_reference_blob_parses_bit_exactly(tmp_path, d, p, n, g, fp32):
    """test_layout.cpp:65-84's round trip, with the B200 library on the import side."""
    if d == 2 and p == 8:
        pytest.skip("the reference's random_field stops at m = 8")
    U = O.ref_random_field(d, p, n, g, fp32, 99)
    path = str(tmp_path / "ref.bin")
    O.ref_export_blob(d, p, n, g, fp32, U, path)
    f = hf.import_blob(path)
    assert (f.d, f.p, f.n_elem, f.group) == (d, p, n, g)
    assert f.precision == (Precision.fp32 if fp32 else Precision.fp64)
    assert np.array_equal(f.data, U)


@ref_only
@pytest.mark.parametrize("d,p,n,g,fp32", SHAPES)
def test_library_blob_is_byte_identical_to_the_reference(tmp_path, d, p, n, g, fp32):
    U = O.random_field(d, p, n, g, fp32, 7)
    prec = Precision.fp32 if fp32 else Precision.fp64
    f = hf.StateField(d, p, n, g, prec, U)
    ours, theirs = str(tmp_path / "ours.bin"), str(tmp_path / "theirs.bin")
    hf.export_blob(f, ours)
    O.ref_export_blob(d, p, n, g, fp32, U, theirs)
    assert _files(ours) == _files(theirs)
    rd, rp, rn, rg, rfp32, data = O.ref_import_blob(ours)
    assert (rd, rp, rn, rg, rfp32) == (d, p, n, g, fp32)
    assert np.array_equal(data, U)


def test_blob_errors_map_to_the_reference_exception_classes(tmp_path):
    f = hf.StateField(3, 2, 6, 4, Precision.fp64, np.arange(hf.StateField(3, 2, 6, 4, 1).total_words(), dtype=float))
    path = str(tmp_path / "x.bin")
    with pytest.raises(HexfuseError, match="missing sidecar"):
        hf.import_blob(path)
    hf.export_blob(f, path)
    g = hf.import_blob(path)
    assert np.array_equal(g.data, f.data)
    side = open(path + ".json").read()
    open(path + ".json", "w").write(side.replace('"fp64"', '"fp16"'))
    with pytest.raises(HexfuseInvalid, match="unknown precision"):  # precision_from_string, core.hpp:16-20
        hf.import_blob(path)
    open(path + ".json", "w").write(side.replace('"words": ', '"words": 1'))
    with pytest.raises(HexfuseError, match="word count mismatch"):
        hf.import_blob(path)
    open(path + ".json", "w").write(side)
    with open(path, "r+b") as fh:
        fh.truncate(100)
    with pytest.raises(HexfuseError, match="short read"):
        hf.import_blob(path)
    open(path + ".json", "w").write("{ not json")
    with pytest.raises(HexfuseError, match="malformed"):
        hf.import_blob(path)
    open(path + ".json", "w").write(side.replace('"words": ', '"words": 99999999999999999999999'))
    with pytest.raises(HexfuseError, match="malformed"):  # no exception escapes the C ABI
        hf.import_blob(path)
    assert not os.path.exists(str(tmp_path / "never.bin.json"))
