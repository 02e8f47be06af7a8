"""CPU: the C-ABI library loads, exports every symbol include/hexfuse_b200.h
declares, and its host-only functions (layout, validation, operators,
selection, partition) agree with the oracle.  No kernel launches here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2107_14027_b200 as hf
from paper_2107_14027_b200 import HexfuseInvalid, Method, PhysParams, Precision, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HF_EINVAL = 2  # include/hexfuse_b200.h
HEADER = os.path.join(ROOT, "include", "hexfuse_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"HF_API\s+[\w\s\*]+?\b(hf_\w+)\s*\(", txt)))


def test_header_symbols_are_exported():
    syms = header_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hf_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    assert sorted(_lib.EXPORTED) == syms
    L = _lib.load()
    for s in syms:
        assert hasattr(L, s)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_torch_in_the_abi():
    code = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)  # declarations only
    assert "torch" not in code.lower()
    assert "std::" not in code and "template" not in code


@pytest.mark.parametrize("d,p,g,n", [(3, 1, 1, 5), (3, 3, 8, 17), (3, 6, 2, 3), (2, 8, 16, 33), (2, 4, 3, 10)])
def test_field_words_and_offsets(d, p, g, n):
    pr = hf.make_problem(d, p, n, g, Precision.fp64, PhysParams())
    assert hf.field_words(pr) == O.field_words(d, p, n, g)
    L = _lib.load()
    m = p + 1
    for e in range(n):
        for v in (0, 1, 1 + d + d * d - 1):
            for (i, j, k) in [(0, 0, 0), (m - 1, 0, m - 1 if d == 3 else 0), (1 % m, m - 1, 0)]:
                assert L.hf_offset(C.byref(pr), e, i, j, k, v) == O.lib().hfo_offset(d, p, g, e, i, j, k, v)


def test_validation_mirrors_reference_errors():
    base = dict(d=3, p=3, n_elem=10, group=4, precision=Precision.fp64, params=PhysParams())
    for kw, msg in [({"d": 4}, "d must"), ({"p": 0}, "p must"), ({"p": 8}, "p must"), ({"group": 0}, "group"),
                    ({"params": PhysParams(nu=-1)}, "nu"), ({"params": PhysParams(zeta=0)}, "zeta"),
                    ({"params": PhysParams(T=0)}, "T must")]:
        a = dict(base)
        a.update(kw)
        pr = hf.make_problem(a["d"], a["p"], a["n_elem"], a["group"], a["precision"], a["params"])
        with pytest.raises(HexfuseInvalid, match=msg):
            hf.validate(pr)
    pr = hf.make_problem(2, 8, 10, 4, Precision.fp32, PhysParams())  # d=2 p=8 is supported (unpinned)
    hf.validate(pr)
    for meth in (Method.planar, Method.planar_managed):
        pr = hf.make_problem(2, 3, 10, 4, Precision.fp32, PhysParams(), method=meth)
        with pytest.raises(HexfuseInvalid, match="planar"):
            hf.validate(pr)  # the reference's planar generator rejects d=2 (codegen_planar.hpp:102)
    pr = hf.make_problem(3, 3, 10, 4, Precision.fp32, PhysParams())
    pr.method = 5  # past HF_METHOD_PLANAR_MANAGED: rejected at the C ABI
    with pytest.raises(HexfuseInvalid, match="unknown method"):
        hf.validate(pr)


def test_derivative_matrix_bitexact_vs_oracle():
    for m in range(2, 10):
        x, D = hf.derivative_matrix(m)
        assert np.array_equal(x, O.gl_nodes(m))
        assert np.array_equal(D, O.derivative_matrix(x))


def test_selection_and_kernel_info_without_device():
    for d, pmax in ((3, 7), (2, 8)):
        for p in range(1, pmax + 1):
            for prec in (Precision.fp32, Precision.fp64):
                pr = hf.make_problem(d, p, 1000, 1, prec, PhysParams())
                meth = hf.selected_method(pr)
                assert meth in (Method.lines, Method.planar)
                info = hf.kernel_info(pr)
                g = hf.preferred_group(pr)
                # group 1 (element-major storage): a one-element chunk when a variant has it,
                # else whole one-element groups per chunk (grouped chunk) -- contiguous either way
                assert g >= 1 and info["bulk_path"]
                assert info["elems_per_cta"] == 1 or info["name"].endswith("_g1"), info["name"]
                assert hf.kernel_info(hf.make_problem(d, p, 1000, g, prec, PhysParams()))["elems_per_cta"] == g
                assert info["shared_bytes"] <= 227 * 1024
                assert info["block_threads"] % 32 == 0
                # with group == elements per CTA every full chunk is one contiguous range: bulk path
                pr2 = hf.make_problem(d, p, 1000, g, prec, PhysParams())
                assert hf.kernel_info(pr2)["bulk_path"]


def test_algorithmic_bytes():
    L = _lib.load()
    pr = hf.make_problem(3, 3, 1, 1, Precision.fp64, PhysParams())
    assert L.hf_algorithmic_bytes_per_point(C.byref(pr)) == 208
    pr = hf.make_problem(3, 3, 1, 1, Precision.fp32, PhysParams())
    assert L.hf_algorithmic_bytes_per_point(C.byref(pr)) == 104
    pr = hf.make_problem(2, 3, 1, 1, Precision.fp32, PhysParams())
    assert L.hf_algorithmic_bytes_per_point(C.byref(pr)) == 56


@pytest.mark.parametrize("n,g,parts", [(1000, 8, 1), (1000, 8, 2), (1001, 8, 4), (7, 4, 8), (2343750, 8, 8)])
def test_partition_covers_every_element_once(n, g, parts):
    pr = hf.make_problem(3, 3, n, g, Precision.fp64, PhysParams())
    gw = g * 64 * 13
    nxt = 0
    for r in range(parts):
        e0, ne, wo = hf.partition(pr, parts, r)
        assert e0 == nxt and e0 % g == 0 and wo == (e0 // g) * gw
        nxt = e0 + ne
    assert nxt == n


def test_unfused_workspace_bytes():
    pr = hf.make_problem(3, 4, 100, 8, Precision.fp32, PhysParams())
    assert hf.unfused_workspace_bytes(pr) == hf.field_words(pr) * 3 * 4


def test_new_entry_points_validate_before_touching_the_device():
    """hf_fr_divergence_faces / hf_fused_divergence_host_batch reject bad arguments
    with HF_EINVAL before any CUDA call (so this runs without a GPU)."""
    L = _lib.load()
    pr = hf.make_problem(3, 3, 10, 2, Precision.fp64, PhysParams())
    assert L.hf_fr_divergence_faces(C.byref(pr), None, None, None, None) == HF_EINVAL
    assert "null buffer" in L.hf_last_error().decode()
    buf = (C.c_double * 4)()
    assert L.hf_fr_divergence_faces(C.byref(pr), buf, buf, buf, None) == HF_EINVAL  # u == divf
    assert "in-place" in L.hf_last_error().decode()
    bad = hf.make_problem(3, 0, 10, 2, Precision.fp64, PhysParams())
    assert L.hf_fr_divergence_faces(C.byref(bad), buf, buf, None, None) == HF_EINVAL
    assert L.hf_fused_divergence_host_batch(None, 1, C.byref(pr), None, None) == HF_EINVAL
    assert "null context" in L.hf_last_error().decode()


def test_fr_residual_validates_mesh_before_any_launch():
    """A mesh whose dims multiply to n_elem but are not all >= 1 is rejected before the
    fused stage-1+2+3+6 kernel runs (so the caller's buffers are untouched)."""
    L = _lib.load()
    pr = hf.make_problem(3, 3, 6, 2, Precision.fp64, PhysParams())
    buf = (C.c_double * 8)()
    out = (C.c_double * 8)()
    for dims in ((-2, -3, 1), (0, 6, 1), (2, 3, 2)):
        d3 = (C.c_int * 3)(*dims)
        assert L.hf_fr_residual(C.byref(pr), d3, buf, buf, out, None) == HF_EINVAL
        assert "dims" in L.hf_last_error().decode()


def test_host_batch_rejects_overlapping_input_and_output():
    """Only exact in-place (u_host == divf_host of the same field) is allowed on the host
    path; partial overlaps are HF_EINVAL before any CUDA call."""
    L = _lib.load()
    pr = hf.make_problem(3, 1, 4, 4, Precision.fp64, PhysParams())
    n = hf.field_words(pr)
    buf = (C.c_double * (2 * n))()
    base = C.addressof(buf)
    us = (C.c_void_p * 1)(base)
    outs = (C.c_void_p * 1)(base + 8 * 16)
    ctx_dummy = C.c_void_p(1)  # never dereferenced: the overlap check comes first
    assert L.hf_fused_divergence_host_batch(ctx_dummy, 1, C.byref(pr), us, outs) == HF_EINVAL
    assert "overlaps" in L.hf_last_error().decode()


def test_overlapping_device_fields_are_rejected_before_launch():
    """u and divf may not share a byte (the kernels read u while other CTAs write divf);
    checked on the addresses alone, before any CUDA call."""
    L = _lib.load()
    pr = hf.make_problem(3, 2, 10, 4, Precision.fp64, PhysParams())
    nbytes = hf.field_words(pr) * 8
    base = 1 << 20
    for off in (0, 8, nbytes - 8):
        assert L.hf_fused_divergence(C.byref(pr), base, base + off, None) == HF_EINVAL
        assert "overlap" in L.hf_last_error().decode()
