"""GPU: the host-buffer path (hf_fused_divergence_host, the (b1) replacement for
oracle_divergence, oracle.hpp:20-62) on fields large enough for the sliced copy
pipeline (ramped slices, three streams), pinned and pageable memory, partial last
group: bit-identical to the device-buffer kernel on the same field, and equal to
the CPU oracle on sampled elements (1e-12 FP64 / 1e-5 FP32)."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import PAR

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,p,fp32,target_mb", [(3, 3, False, 400), (3, 6, True, 300), (2, 2, True, 60),
                                                (3, 1, False, 5)])
def test_host_path_matches_device_path(cuda, d, p, fp32, target_mb):
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    prec = Precision.fp32 if fp32 else Precision.fp64
    w = 4 if fp32 else 8
    g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
    nv, npt = O.n_vars(d), (p + 1) ** d
    n = max(g, int(target_mb * 2 ** 20 / (nv * npt * w)) // g * g) + 1  # partial last group
    pr = hf.make_problem(d, p, n, g, prec, PAR, with_source=True)
    dt = torch.float32 if fp32 else torch.float64
    gen = torch.Generator().manual_seed(5)
    u = (torch.rand(hf.field_words(pr), generator=gen, dtype=torch.float64) * 2 - 1).to(dt)
    # padding elements of the last group stay zero, as in a StateField
    nwg = hf.field_words(pr) // ((n + g - 1) // g)
    last = u[-nwg:].view(nv * npt, g)
    last[:, n % g:] = 0
    # device path
    ud = u.cuda()
    od = torch.zeros_like(ud)
    hf.fused_divergence_device(pr, ud, od)
    torch.cuda.synchronize()
    ref = od.cpu()
    ctx = hf.Context(0)
    for pinned in (True, False):
        src = u.pin_memory() if pinned else u.clone()
        dst = torch.zeros_like(src)
        if pinned:
            dst = dst.pin_memory()
        ctx.run(pr, src, dst)
        assert torch.equal(dst, ref), f"host path differs from the device path (pinned={pinned})"
    ctx.close()
    # oracle on a sample: the first and the last (partial) group
    U = u.double().numpy()
    for e0, e1 in ((0, min(n, g)), ((n - 1) // g * g, n)):
        out = np.zeros_like(U)
        O.oracle_divergence_elements(d, p, g, U, out, PAR.nu, PAR.zeta, PAR.T, (1.0, 1.0, 1.0), True, e0, e1)
        sl = slice(e0 // g * nwg, ((e1 + g - 1) // g) * nwg)
        got = ref.double().numpy()[sl]
        want = out[sl]
        err = np.max(np.abs(got - want)) / max(1.0, np.max(np.abs(want)))
        assert err <= (1e-5 if fp32 else 1e-12), err


def test_host_batch_matches_device_path(cuda):
    """hf_fused_divergence_host_batch: several fields (mixed d, p, precision, a partial
    last group, an empty field) through one copy pipeline, each bit-identical to the
    device-buffer kernel on the same field."""
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    specs = [(3, 1, True, 120), (3, 6, False, 90), (2, 4, True, 40), (3, 3, False, 0), (3, 3, False, 150)]
    gen = torch.Generator().manual_seed(11)
    items, refs = [], []
    for d, p, fp32, target_mb in specs:
        prec = Precision.fp32 if fp32 else Precision.fp64
        g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
        nv, npt, w = O.n_vars(d), (p + 1) ** d, (4 if fp32 else 8)
        n = 0 if target_mb == 0 else max(g, int(target_mb * 2 ** 20 / (nv * npt * w)) // g * g) + 1
        pr = hf.make_problem(d, p, n, g, prec, PAR, with_source=True)
        dt = torch.float32 if fp32 else torch.float64
        u = (torch.rand(hf.field_words(pr), generator=gen, dtype=torch.float64) * 2 - 1).to(dt)
        if n:
            nwg = hf.field_words(pr) // ((n + g - 1) // g)
            u[-nwg:].view(nv * npt, g)[:, n % g:] = 0  # padding elements stay zero
            ud = u.cuda()
            od = torch.zeros_like(ud)
            hf.fused_divergence_device(pr, ud, od)
            torch.cuda.synchronize()
            refs.append(od.cpu())
        else:
            refs.append(u.clone())
        src = u.pin_memory()
        dst = torch.zeros_like(src).pin_memory() if n else src.clone()
        items.append((pr, src, dst))
    ctx = hf.Context(0)
    ctx.run_batch(items)
    ctx.close()
    for (pr, src, dst), ref in zip(items, refs):
        if pr.n_elem:
            assert torch.equal(dst, ref), (pr.d, pr.p, pr.precision)


@pytest.mark.parametrize("pinned", [True, False])
def test_host_path_in_place(cuda, pinned):
    """u_host == divf_host: the result overwrites the input, equal to the out-of-place run."""
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    d, p = 3, 3
    g = hf.preferred_group(hf.make_problem(d, p, 1, 1, Precision.fp64, PAR))
    n = int(60 * 2 ** 20 / (13 * 64 * 8)) // g * g
    pr = hf.make_problem(d, p, n, g, Precision.fp64, PAR, with_source=True)
    gen = torch.Generator().manual_seed(9)
    u = torch.rand(hf.field_words(pr), generator=gen, dtype=torch.float64) * 2 - 1
    ctx = hf.Context(0)
    ref = torch.zeros_like(u)
    ctx.run(pr, u.clone(), ref)
    buf = u.clone().pin_memory() if pinned else u.clone()
    ctx.run(pr, buf, buf)
    ctx.close()
    assert torch.equal(buf, ref)


@pytest.mark.parametrize("fp32", [False, True])
def test_blob_in_divergence_blob_out(cuda, tmp_path, fp32):
    """hf_fused_divergence_blob: a blob the reference's export_blob wrote (or the library's
    byte-identical one where the reference is absent) -> the B200 host path -> a result
    blob equal to the oracle's divergence."""
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    d, p, n, g = 3, 3, 45, 32
    U = O.random_field(d, p, n, g, fp32, 31)
    src = str(tmp_path / "u.bin")
    if O.ref_available():
        O.ref_export_blob(d, p, n, g, fp32, U, src)
    else:
        hf.export_blob(hf.StateField(d, p, n, g, Precision.fp32 if fp32 else Precision.fp64, U), src)
    dst = str(tmp_path / "div.bin")
    hf.fused_divergence_blob(src, dst, PAR, (1.0, 0.5, 2.0), with_source=True)
    out = hf.import_blob(dst)
    assert (out.d, out.p, out.n_elem, out.group) == (d, p, n, g)
    ref = O.oracle_divergence(d, p, n, g, U, PAR.nu, PAR.zeta, PAR.T, (1.0, 0.5, 2.0), True)
    assert O.field_rel_error(d, p, n, g, out.data, ref) <= (1e-5 if fp32 else 1e-12)
    real = np.broadcast_to((np.arange(g) < n - g)[None, :], (13 * 64, g)).reshape(-1)
    assert np.all(out.data[-13 * 64 * g:][~real] == 0.0)  # padding of the partial group comes back zero
