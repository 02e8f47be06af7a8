"""GPU parity of the mapped-element kernel (non-constant Jacobian):
hf_fused_divergence_mapped vs the CPU oracle's mapped restatement
(oracle/hexfuse_oracle.c, hfo_oracle_divergence_mapped), which is pinned to the
compiled reference on axis-aligned boxes (tests/test_oracle.py).  Tolerances are
the north star's: 1e-12 relative FP64, 1e-5 FP32 (verify.hpp:19-35 metric)."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import PAR, padding_mask

pytestmark = pytest.mark.gpu


def run_mapped(d, p, n, group, fp32, U, G, params=PAR, with_source=False):
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    dt = torch.float32 if fp32 else torch.float64
    pr = hf.make_problem(d, p, n, group, Precision.fp32 if fp32 else Precision.fp64, params,
                         with_source=with_source)
    assert hf.field_words(pr) == U.size and hf.geometry_words(pr) == G.size
    u = torch.from_numpy(U).to(dt).cuda()
    g = torch.from_numpy(G).to(dt).cuda()
    o = torch.full_like(u, 7.25)
    hf.fused_divergence_mapped_device(pr, u, g, o)
    torch.cuda.synchronize()
    return o.double().cpu().numpy()


def check_mapped(d, p, n, group, fp32, U, G, params=PAR, with_source=False):
    got = run_mapped(d, p, n, group, fp32, U, G, params, with_source)
    ref = O.oracle_divergence_mapped(d, p, n, group, U, G, params.nu, params.zeta, params.T, with_source)
    err = O.field_rel_error(d, p, n, group, got, ref)
    tol = 1e-5 if fp32 else 1e-12
    assert err <= tol, f"mapped d={d} p={p} n={n} group={group} fp32={fp32} src={with_source}: {err:.3e}"
    real = padding_mask(d, p, n, group)
    assert np.all(got[~real] == 7.25), "kernel wrote into padding elements"
    return err


def _ne(d, p, fp32):
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import PhysParams, Precision
    return hf.mapped_kernel_info(hf.make_problem(d, p, 1, 1, Precision.fp32 if fp32 else Precision.fp64,
                                                 PhysParams()))["elems_per_cta"]


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("d,p", [(3, 1), (3, 2), (3, 3), (3, 4), (3, 5), (3, 6), (3, 7),
                                 (2, 1), (2, 3), (2, 5), (2, 8)])
def test_mapped_curved_random(cuda, d, p, fp32):
    g = _ne(d, p, fp32)
    n = 2 * g + 1  # bulk chunks + a partial last group
    for t, src in enumerate([False, True]):
        U = O.random_field(d, p, n, g, fp32, 900 + p + t)
        G = O.random_geometry(d, n, g, 31 + t, amp=0.2, fp32=fp32)
        check_mapped(d, p, n, g, fp32, U, G, with_source=src)


@pytest.mark.parametrize("group", [1, 3, 8, 64])
def test_mapped_layouts_fp64_p3(cuda, group):
    n = 37
    U = O.random_field(3, 3, n, group, False, 5)
    G = O.random_geometry(3, n, group, 5)
    check_mapped(3, 3, n, group, False, U, G, with_source=True)


@pytest.mark.parametrize("d,p", [(3, 2), (3, 4), (2, 3)])
def test_mapped_boxes_equal_constant_jacobian_kernel(cuda, d, p):
    """Axis-aligned boxes: the mapped kernel equals the reference's constant-Jacobian
    result with jac = 1/h (oracle_divergence, pinned bit-exactly to the reference)."""
    from gpu_util import run_device
    h = (0.5, 0.7, 0.9)
    g = _ne(d, p, False)
    n = 3 * g
    U = O.random_field(d, p, n, g, False, 77)
    G = O.box_geometry(d, n, g, h)
    got = run_mapped(d, p, n, g, False, U, G, with_source=True)
    jac = tuple(1.0 / x for x in h)
    ref = O.oracle_divergence(d, p, n, g, U, PAR.nu, PAR.zeta, PAR.T, jac, True)
    assert O.field_rel_error(d, p, n, g, got, ref) <= 1e-12
    lines = run_device(d, p, n, g, False, U, jac=jac, with_source=True)
    assert O.field_rel_error(d, p, n, g, got, lines) <= 1e-12


@pytest.mark.parametrize("fp32", [False, True])
def test_mapped_freestream(cuda, fp32):
    """Constant state on curved elements: zero divergence (discrete metric identity, p >= 2)."""
    d, p = 3, 3
    g = _ne(d, p, fp32)
    n = 2 * g
    nv = O.n_vars(d)
    U = np.zeros(O.field_words(d, p, n, g)).reshape(-1, nv, (p + 1) ** d, g)
    for v in range(nv):
        U[:, v] = 0.3 + 0.05 * v
    G = O.random_geometry(d, n, g, 3, amp=0.2, fp32=fp32)
    got = run_mapped(d, p, n, g, fp32, U.reshape(-1), G, params=PAR)
    assert np.max(np.abs(got)) < (2e-4 if fp32 else 1e-11)
