"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle
restatement (oracle/hexfuse_oracle.c, itself pinned bit-exactly to the
reference).  Tolerances: 1e-12 relative for FP64 and 1e-5 for FP32 in the
reference's field_rel_error metric (verify.hpp:19-35; BASELINE north star).
Seeds and physical parameters follow acceptance.cpp:46-52 (seed 2024,
nu = 1/1600) and test_oracle.cpp:134-165 (jac {1,0.5,2}, alternating source)."""
import numpy as np
import pytest

import oracle as O
from paper_2107_14027_b200 import Method, PhysParams

pytestmark = pytest.mark.gpu

from gpu_util import PAR, check_parity, run_device  # noqa: E402


def _field(d, p, n, group, fp32, seed):
    return O.random_field(d, p, n, group, fp32, seed)


# ---------------------------------------------------------------- lines (default) method, all orders
@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
def test_lines_d3_random(cuda, p, fp32):
    import paper_2107_14027_b200 as hf
    g = hf.preferred_group(hf.make_problem(3, p, 1, 1, int(not fp32), PAR, method=Method.lines))
    n = 3 * g + 1  # full bulk chunks plus a partial last group
    for t, src in enumerate([False, True]):
        U = _field(3, p, n, g, fp32, 2024 + t)
        check_parity(3, p, n, g, fp32, U, with_source=src, method=Method.lines)


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_lines_d2_random(cuda, p, fp32):
    import paper_2107_14027_b200 as hf
    g = hf.preferred_group(hf.make_problem(2, p, 1, 1, int(not fp32), PAR, method=Method.lines))
    n = 2 * g + 3
    for t, src in enumerate([False, True]):
        U = _field(2, p, n, g, fp32, 77 + t)
        check_parity(2, p, n, g, fp32, U, with_source=src, jac=(1.0, 2.0, 0.0), method=Method.lines)


# ---------------------------------------------------------------- non-unit metric (test_oracle.cpp:134-146)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_nonunit_jac_fp64(cuda, p):
    par = PhysParams(3e-3, 2.5, 1.0)
    for t in range(3):
        U = _field(3, p, 37, 4, False, 100 + 10 * p + t)
        for method in (Method.lines, Method.planar, Method.planar_managed, Method.unfused):
            check_parity(3, p, 37, 4, False, U, params=par, jac=(1.0, 0.5, 2.0), with_source=(t % 2 == 0),
                         method=method)


# ---------------------------------------------------------------- every layout path of the lines kernel
@pytest.mark.parametrize("group", [1, 2, 3, 5, 8, 16, 32, 64])
def test_lines_groups_fp64_p3(cuda, group):
    U = _field(3, 3, 70, group, False, 5)
    check_parity(3, 3, 70, group, False, U, with_source=True, method=Method.lines)


@pytest.mark.parametrize("group", [1, 4, 6, 16, 32, 48])
def test_lines_groups_fp32_p4(cuda, group):
    U = _field(3, 4, 50, group, True, 6)
    check_parity(3, 4, 50, group, True, U, method=Method.lines)


def test_lines_misaligned_pointer(cuda):
    # a base pointer that is not 16-byte aligned must fall back to the guarded path
    U = _field(3, 2, 64, 16, False, 9)
    check_parity(3, 2, 64, 16, False, U, method=Method.lines, offset_bytes=8)


@pytest.mark.parametrize("variant", list(range(28)))
@pytest.mark.parametrize("d,p,fp32", [(3, 1, True), (3, 3, False), (3, 3, True), (3, 4, True), (3, 6, False),
                                      (3, 6, True), (2, 3, True), (2, 7, True), (2, 8, True)])
def test_lines_variants(cuda, d, p, fp32, variant):
    """Every lines variant (3..6 = persistent TMA-ring kernel), bulk chunks + guarded tail, +-source."""
    import paper_2107_14027_b200 as hf
    pr = hf.make_problem(d, p, 1, 1, int(not fp32), PAR)
    try:
        info = hf.variant_info(pr, Method.lines, variant)
    except hf.HexfuseInvalid:
        pytest.skip("variant not instantiated for this order")
    g = info["elems_per_cta"]
    # contiguous chunks (group == NE, any alignment; with and without a partial last group),
    # row-mode chunks (group = 2 NE, 4 NE)
    for n, group, src in [(5 * g + 1, g, False), (6 * g, g, True), (7 * g, 2 * g, True), (3 * g + 2, 4 * g, True)]:
        U = _field(d, p, n, group, fp32, 11 + n)
        got = run_device(d, p, n, group, fp32, U, method=Method.lines, variant=variant, with_source=src)
        ref = O.oracle_divergence(d, p, n, group, U, PAR.nu, PAR.zeta, PAR.T, (1.0, 1.0, 1.0), src)
        err = O.field_rel_error(d, p, n, group, got, ref)
        assert err <= (1e-5 if fp32 else 1e-12), (n, group, src, err)


@pytest.mark.parametrize("d,p,fp32", [(3, 4, False), (3, 2, True), (3, 5, False), (3, 6, False), (3, 7, True), (2, 6, False)])
def test_component_split_is_bit_identical(cuda, d, p, fp32):
    """The component-split variants (19-23: d threads per line) run the same arithmetic in the
    same order as their one-thread-per-line counterparts (0, 1, 2, 7, 3): equal bit for bit."""
    import paper_2107_14027_b200 as hf
    pr0 = hf.make_problem(d, p, 1, 1, int(not fp32), PAR)
    pairs = [(19, 0), (20, 1), (21, 2), (22, 7), (23, 3)]
    ran = 0
    for cs, base in pairs:
        try:
            g = hf.variant_info(pr0, Method.lines, cs)["elems_per_cta"]
            assert hf.variant_info(pr0, Method.lines, base)["elems_per_cta"] == g
        except hf.HexfuseInvalid:
            continue
        n = 37 * g + 1
        U = _field(d, p, n, g, fp32, 600 + cs)
        for src in (False, True):
            a = run_device(d, p, n, g, fp32, U, method=Method.lines, variant=cs, with_source=src)
            b = run_device(d, p, n, g, fp32, U, method=Method.lines, variant=base, with_source=src)
            assert np.array_equal(a, b), (cs, base, src)
        ran += 1
    if not ran:
        pytest.skip("no component-split variant instantiated (production build)")


def test_pipe_many_chunks_per_cta(cuda):
    """More chunks than resident CTAs: every CTA cycles its stage ring several times."""
    import paper_2107_14027_b200 as hf
    for fp32, p in [(False, 3), (True, 5)]:
        pr = hf.make_problem(3, p, 1, 1, int(not fp32), PAR)
        for variant in (3, 4, 5, 6, 8, 9, 10, 11, 12, 13, 14, 15, 23):
            try:
                g = hf.variant_info(pr, Method.lines, variant)["elems_per_cta"]
            except hf.HexfuseInvalid:
                continue
            n = g * 148 * 9 + 3
            U = _field(3, p, n, g, fp32, 5)
            got = run_device(3, p, n, g, fp32, U, method=Method.lines, variant=variant)
            ref = O.oracle_divergence(3, p, n, g, U, PAR.nu, PAR.zeta, PAR.T)
            assert O.field_rel_error(3, p, n, g, got, ref) <= (1e-5 if fp32 else 1e-12)


# ---------------------------------------------------------------- planar method (d = 3)
@pytest.mark.parametrize("method", [Method.planar, Method.planar_managed])
@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_planar_random(cuda, p, fp32, method):
    for t, src in enumerate([False, True]):
        U = _field(3, p, 45, 32, fp32, 2024 + t)
        check_parity(3, p, 45, 32, fp32, U, with_source=src, method=method)


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_planar_managed_layouts(cuda, p, fp32):
    """Managed planar (every operand resident in shared memory): bulk-staged chunks
    (group == elements per CTA, any alignment), row-mode chunks, group 1 / 3 (guarded
    staging), a partial last chunk, and the same numbers as the unmanaged planar kernel
    (same accumulation order, codegen_planar.hpp:97-210)."""
    import paper_2107_14027_b200 as hf
    g = hf.variant_info(hf.make_problem(3, p, 1, 1, int(not fp32), PAR), Method.planar_managed, 0)["elems_per_cta"]
    for n, group, src in [(3 * g + 1, g, True), (4 * g, 2 * g, False), (2 * g + 1, 1, True), (2 * g + 2, 3, False)]:
        U = _field(3, p, n, group, fp32, 300 + n + group)
        got = check_parity(3, p, n, group, fp32, U, with_source=src, method=Method.planar_managed)
        assert got <= (1e-5 if fp32 else 1e-12)
    U = _field(3, p, 2 * g, g, fp32, 17)
    a = run_device(3, p, 2 * g, g, fp32, U, method=Method.planar_managed, with_source=True)
    b = run_device(3, p, 2 * g, g, fp32, U, method=Method.planar, with_source=True)
    assert O.field_rel_error(3, p, 2 * g, g, a, b) <= (1e-6 if fp32 else 1e-14)


# ---------------------------------------------------------------- unfused comparator
@pytest.mark.parametrize("d,p", [(3, 1), (3, 3), (3, 4), (3, 6), (2, 2), (2, 8)])
@pytest.mark.parametrize("fp32", [False, True])
def test_unfused_random(cuda, d, p, fp32):
    for t, src in enumerate([False, True]):
        U = _field(d, p, 40, 8, fp32, 31 + t)
        check_parity(d, p, 40, 8, fp32, U, with_source=src, method=Method.unfused)


# ---------------------------------------------------------------- deterministic vortex fixture (verify.hpp:85-91)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("fp32", [False, True])
def test_tgv_fixture(cuda, p, fp32):
    import paper_2107_14027_b200 as hf
    g = hf.preferred_group(hf.make_problem(3, p, 1, 1, int(not fp32), PAR))
    n = 64
    U = O.tgv_field(p, n, g, fp32)
    for method in (Method.auto, Method.planar, Method.planar_managed):
        check_parity(3, p, n, g, fp32, U, method=method)


# ---------------------------------------------------------------- analytic known answers (test_oracle.cpp:90-132)
def test_constant_field_zero_divergence(cuda):
    from gpu_util import padding_mask
    d, p, n, g = 3, 2, 3, 2
    U = np.zeros(O.field_words(d, p, n, g)).reshape(-1, 13, 27, g)
    for v in range(13):
        U[:, v, :, :] = 0.5 + 0.1 * v
    U = U.reshape(-1)
    real = padding_mask(d, p, n, g).reshape(-1, 13, 27, g)
    for method in (Method.lines, Method.planar, Method.planar_managed, Method.unfused):
        got = run_device(d, p, n, g, False, U, method=method).reshape(-1, 13, 27, g)
        assert np.max(np.abs(got[real])) < 1e-12
        src = run_device(d, p, n, g, False, U, with_source=True, method=method).reshape(-1, 13, 27, g)
        for v in range(13):
            want = -(0.5 + 0.1 * v) if v >= 4 else 0.0
            sel = src[:, v][real[:, v]]
            assert np.max(np.abs(sel - want)) < 1e-12


def test_linear_velocity_exact(cuda):
    par = PhysParams(1e-2, 2.5, 0.5)
    for p in (2, 3):
        m = p + 1
        nodes = O.gl_nodes(m)
        U = np.zeros(O.field_words(3, p, 1, 1))
        for k in range(m):
            for j in range(m):
                for i in range(m):
                    U[i + m * j + m * m * k + m ** 3 * 1] = nodes[i]  # u = x
        for method in (Method.lines, Method.planar, Method.planar_managed, Method.unfused):
            got = run_device(3, p, 1, 1, False, U, params=par, method=method)
            for k in range(m):
                for j in range(m):
                    for i in range(m):
                        pt = i + m * j + m * m * k
                        assert abs(got[pt] - (-par.zeta)) < 1e-10 * par.zeta
                        assert abs(got[pt + m ** 3] - (-2.0 * nodes[i])) < 1e-10
                        assert abs(got[pt + 4 * m ** 3] - (1.0 / par.T)) < 1e-10 / par.T


# ---------------------------------------------------------------- config 1 at full size (32768 x p3 fp64)
def test_config1_full_oracle(cuda):
    """BASELINE config 1: d=3 p=3 FP64, 32768 elements, seed 2024, the whole field vs the oracle."""
    import paper_2107_14027_b200 as hf
    g = hf.preferred_group(hf.make_problem(3, 3, 1, 1, 1, PAR))
    U = _field(3, 3, 32768, g, False, 2024)
    err = check_parity(3, 3, 32768, g, False, U, with_source=False)
    assert err <= 1e-12
    err = check_parity(3, 3, 32768, g, False, U, with_source=True)
    assert err <= 1e-12


# ---------------------------------------------------------------- empty problems (n_elem = 0)
def test_empty_problems_are_no_ops(cuda):
    """n_elem = 0 on every entry point: success, nothing launched, nothing written
    (the reference's oracle returns an empty field for an empty input)."""
    import torch
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Method, Precision
    for d, p in ((3, 3), (2, 5)):
        for prec in (Precision.fp32, Precision.fp64):
            pr = hf.make_problem(d, p, 0, 4, prec, PAR, with_source=True)
            assert hf.field_words(pr) == 0
            buf = torch.full((8,), 3.5, device="cuda", dtype=torch.float64)
            hf.fused_divergence_device(pr, buf, buf[4:])
            for meth in (Method.lines, Method.unfused) if d == 2 else (Method.lines, Method.planar,
                                                                     Method.planar_managed, Method.unfused):
                pr.method = int(meth)
                if meth == Method.unfused:
                    hf.unfused_divergence_device(pr, buf, buf[4:], buf[2:])
                else:
                    hf.fused_divergence_device(pr, buf, buf[4:])
            pr.method = int(Method.auto)
            hf.fused_divergence_mapped_device(pr, buf, buf[2:], buf[4:])
            hf.fr_project_device(pr, buf, buf[4:])
            torch.cuda.synchronize()
            assert torch.all(buf == 3.5)
            U = hf.StateField(d, p, 0, 4, prec)
            out = hf.fused_divergence(U, PAR, with_source=True)
            assert out.n_elem == 0 and out.data.size == 0


# ---------------------------------------------------------------- caller-chosen AoSoA groups (tile mode)
# The reference's own groups: planar 4*floor(32/m) (p1 64, p2 40, p3 32, p4 24, p5 20, p6 16)
# and the preset lines blocks (fp64 p3 192/16 = 12, p4 200/25 = 8; layout.hpp:76-85,
# presets.hpp:25-37), plus odd groups whose stride rules TMA out (guarded path).
@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_caller_groups_d3(cuda, p, fp32):
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    groups = sorted({64, 40, 32, 24, 20, 16, 12, 8, 4 * (32 // (p + 1)), 15, 5, 4, 2, 1})
    for gi, g in enumerate(groups):
        n = 2 * g + (g // 2 + 1) + 150  # full chunks of every chunk size + a partial last group
        U = _field(3, p, n, g, fp32, 4000 + 10 * p + gi)
        check_parity(3, p, n, g, fp32, U, with_source=(gi % 2 == 0))
    pr = hf.make_problem(3, p, 100, 40, Precision.fp32 if fp32 else Precision.fp64, PAR)
    name = hf.kernel_info(pr)["name"]
    assert "_tile" in name or "ne40" in name, name


@pytest.mark.parametrize("fp32", [False, True])
def test_tile_ring_caller_groups_d3_p5(cuda, fp32):
    """The tile ring (lines variant 24: two-stage TMA ring, one tensor copy per chunk and
    direction) with several chunks per CTA -- the ring's refill path -- for whole groups and a
    partial last group; forced on groups that leave the last sub-chunk of every group short
    (12, 20: zero-filled and clipped by the tensor maps)."""
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    prec = Precision.fp32 if fp32 else Precision.fp64
    for gi, g in enumerate((8, 16, 32, 64, 4 if not fp32 else 8)):
        n = (3 * 148 * 8 // g) * g + g // 2 + 3
        pr = hf.make_problem(3, 5, n, g, prec, PAR)
        assert hf.kernel_info(pr)["name"].startswith("hf_lines_pipe_d3_p5"), hf.kernel_info(pr)["name"]
        U = _field(3, 5, n, g, fp32, 7000 + gi)
        check_parity(3, 5, n, g, fp32, U, with_source=(gi % 2 == 1))
    for gi, g in enumerate((12, 20)):
        n = (3 * 148 * 8 // g) * g + 5
        U = _field(3, 5, n, g, fp32, 7100 + gi)
        check_parity(3, 5, n, g, fp32, U, method=Method.lines, variant=24, with_source=(gi == 0))


@pytest.mark.parametrize("p", [1, 3, 5, 8])
def test_caller_groups_d2(cuda, p):
    for gi, g in enumerate((12, 24, 40, 64, 7, 1, 2, 4)):
        n = 3 * g + 2 + 260
        for fp32 in (True, False):
            U = _field(2, p, n, g, fp32, 6000 + p + gi)
            check_parity(2, p, n, g, fp32, U, with_source=fp32, jac=(1.0, 0.5, 0.0))


def test_tile_mode_with_misaligned_buffers_takes_the_guarded_path(cuda):
    """An 8-byte offset (not 16) rules TMA out: same results through the guarded path."""
    U = _field(3, 3, 70, 32, False, 8)
    check_parity(3, 3, 70, 32, False, U, offset_bytes=8)


@pytest.mark.parametrize("d,p,fp32", [(3, 3, False), (3, 3, True), (3, 7, True), (2, 7, True)])
def test_padded_chunks_edge_cases(cuda, d, p, fp32):
    """The selected padded-chunk kernels (lines variants 25-27, TMA box wider than the row /
    plane): a partial last chunk (guarded path into the padded layout), a misaligned base
    (falls back to the unpadded chunk) and a caller group that is not the chunk."""
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    prec = Precision.fp32 if fp32 else Precision.fp64
    g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
    assert hf.kernel_info(hf.make_problem(d, p, 10 * g, g, prec, PAR))["name"].endswith("_xp")
    n = 37 * g + max(1, g // 2)
    U = _field(d, p, n, g, fp32, 8100 + p)
    check_parity(d, p, n, g, fp32, U, with_source=True)
    check_parity(d, p, n, g, fp32, U, offset_bytes=8)
    U2 = _field(d, p, n, 2 * g, fp32, 8200 + p)
    check_parity(d, p, n, 2 * g, fp32, U2)


# ---------------------------------------------------------------- stream order under programmatic dependent launch
@pytest.mark.parametrize("d,p,fp32", [(3, 3, False), (3, 6, False), (2, 2, True), (3, 1, True)])
def test_dependent_back_to_back_launches(cuda, d, p, fp32):
    """The fused kernels are launched with programmatic dependent launch (hf_launch.cuh
    launch_kernel): a launch may start while the previous kernel drains, and waits
    (griddepcontrol.wait) before touching HBM.  Chain u -> o1 -> o2 -> o3 back to back with
    no host synchronisation: each stage must read its predecessor's finished output."""
    import torch
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    prec = Precision.fp32 if fp32 else Precision.fp64
    g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
    n = 40 * g + 3
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    pr = hf.make_problem(d, p, n, g, prec, par)
    U = _field(d, p, n, g, fp32, 4242)
    dt = torch.float32 if fp32 else torch.float64
    bufs = [torch.from_numpy(U).to(dt).cuda()] + [torch.zeros(U.size, dtype=dt, device="cuda") for _ in range(3)]
    for k in range(3):
        hf.fused_divergence_device(pr, bufs[k], bufs[k + 1])
    torch.cuda.synchronize()
    ref = U
    for k in range(3):
        # the device computes each stage from the previous stage's rounded output
        ref_in = bufs[k].double().cpu().numpy()
        ref = O.oracle_divergence(d, p, n, g, ref_in, par.nu, par.zeta, par.T)
        err = O.field_rel_error(d, p, n, g, bufs[k + 1].double().cpu().numpy(), ref)
        assert err <= (1e-5 if fp32 else 1e-12), f"stage {k + 1}: {err:.3e}"


def test_cuda_graph_capture_and_replay(cuda):
    """The launch path is capture-safe (no host synchronisation, no allocation; the
    programmatic-dependent-launch attribute becomes a graph edge): launches captured into
    a CUDA graph replay to the same bits as stream launches, for the one-chunk, the TMA-ring,
    the component-split and the tile-mode kernels."""
    import torch
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    cases = []
    for d, p, prec, g in [(3, 3, Precision.fp64, None), (3, 6, Precision.fp64, None), (3, 4, Precision.fp64, None),
                          (3, 2, Precision.fp32, 24), (2, 5, Precision.fp32, None)]:
        g = g or hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
        n = 20 * g + 1
        pr = hf.make_problem(d, p, n, g, prec, PAR, with_source=True)
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        u = torch.empty(hf.field_words(pr), dtype=dt, device="cuda").uniform_(-1, 1)
        cases.append((pr, u, torch.zeros_like(u), torch.zeros_like(u)))
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for pr, u, o, _ in cases:
            hf.fused_divergence_device(pr, u, o, st)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for pr, u, _, og in cases:
            hf.fused_divergence_device(pr, u, og, st)
    with torch.cuda.stream(st):
        graph.replay()
    torch.cuda.synchronize()
    for pr, u, o, og in cases:
        assert torch.equal(o, og), hf.kernel_info(pr)["name"]
