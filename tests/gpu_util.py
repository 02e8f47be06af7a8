"""Helpers shared by the GPU parity tests: run the B200 kernels through the C ABI
on a field, and compare with the CPU oracle (oracle/, test infrastructure)."""
import numpy as np
import torch

import oracle as O
import paper_2107_14027_b200 as hf
from paper_2107_14027_b200 import Method, PhysParams, Precision

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)  # acceptance.cpp:52


def run_device(d, p, n_elem, group, fp32, U, params=PAR, jac=(1.0, 1.0, 1.0), with_source=False,
               method=Method.auto, variant=None, offset_bytes=0):
    """Run one kernel on the field U (float64 numpy, AoSoA) and return the result as float64 numpy.
    The output buffer is pre-filled with a sentinel so that writes to padding are detected."""
    dt = torch.float32 if fp32 else torch.float64
    pr = hf.make_problem(d, p, n_elem, group, Precision.fp32 if fp32 else Precision.fp64, params, jac,
                         with_source, method)
    words = hf.field_words(pr)
    assert words == U.size
    pad = offset_bytes // (4 if fp32 else 8)
    ubuf = torch.zeros(words + pad, dtype=dt, device="cuda")
    ubuf[pad:] = torch.from_numpy(U).to(dt)
    obuf = torch.full((words + pad,), 7.25, dtype=dt, device="cuda")
    u = ubuf[pad:]
    o = obuf[pad:]
    if method == Method.unfused:
        ws = torch.empty(hf.unfused_workspace_bytes(pr) // u.element_size(), dtype=dt, device="cuda")
        hf.unfused_divergence_device(pr, u, o, ws)
    elif variant is not None:
        hf.fused_divergence_variant(pr, method if method != Method.auto else Method.lines, variant, u, o)
    else:
        hf.fused_divergence_device(pr, u, o)
    torch.cuda.synchronize()
    return o.double().cpu().numpy()


def padding_mask(d, p, n_elem, group):
    nv, npt = 1 + d + d * d, (p + 1) ** d
    ng = (n_elem + group - 1) // group
    real = (np.arange(ng * group).reshape(ng, group) < n_elem)[:, None, None, :]
    return np.broadcast_to(real, (ng, nv, npt, group)).reshape(-1)


def check_parity(d, p, n_elem, group, fp32, U, tol=None, **kw):
    got = run_device(d, p, n_elem, group, fp32, U, **kw)
    params = kw.get("params", PAR)
    ref = O.oracle_divergence(d, p, n_elem, group, U, params.nu, params.zeta, params.T,
                              kw.get("jac", (1.0, 1.0, 1.0)), kw.get("with_source", False))
    err = O.field_rel_error(d, p, n_elem, group, got, ref)
    if tol is None:
        tol = 1e-5 if fp32 else 1e-12
    assert err <= tol, f"d={d} p={p} n={n_elem} group={group} fp32={fp32} {kw}: rel err {err:.3e} > {tol:.0e}"
    # padding elements are neither read nor written (render.hpp:95,102)
    real = padding_mask(d, p, n_elem, group)
    assert np.all(got[~real] == 7.25), "kernel wrote into padding elements"
    return err
