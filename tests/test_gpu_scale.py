"""GPU parity at the BASELINE sizes (configs 2, 3 and 5): the selected kernel runs over the
whole field, and sampled element groups are compared with the CPU oracle
(oracle_divergence, oracle.hpp:20-62, restated in oracle/hexfuse_oracle.c) -- the first
and last group, the groups holding byte offset 2^32 and word index 2^31 (config 5's
15.6 GB fields), and random groups spread over the field ("a sampled
subset of element groups for configs 3 and 5").  Tolerances 1e-12 (FP64) / 1e-5 (FP32)
in the field_rel_error metric (verify.hpp:19-33)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

from gpu_util import PAR  # noqa: E402

SENTINEL = 7.25


def _sampled_parity(d, p, n_elem, fp32, with_source, n_random, seed):
    import torch

    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    prec = Precision.fp32 if fp32 else Precision.fp64
    g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
    pr = hf.make_problem(d, p, n_elem, g, prec, PAR, with_source=with_source)
    dt = torch.float32 if fp32 else torch.float64
    words = hf.field_words(pr)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    u = torch.empty(words, dtype=dt, device="cuda")
    u.uniform_(-1.0, 1.0, generator=gen)
    o = torch.full((words,), SENTINEL, dtype=dt, device="cuda")
    hf.fused_divergence_device(pr, u, o)
    torch.cuda.synchronize()

    nv, npt = 1 + d + d * d, (p + 1) ** d
    gw = g * npt * nv
    wb = u.element_size()
    n_groups = -(-n_elem // g)
    pick = {0, n_groups - 1}
    for boundary_word in (2 ** 32 // wb, 2 ** 31):  # byte offset 2^32, word index 2^31
        if boundary_word < words:
            gi = boundary_word // gw
            pick |= {gi, min(n_groups - 1, gi + 1)}
    rng = np.random.default_rng(seed)
    pick |= set(int(x) for x in rng.integers(0, n_groups, size=n_random))
    maxdiff = maxref = 0.0
    for gi in sorted(pick):
        n_e = min(g, n_elem - gi * g)
        U = u[gi * gw:(gi + 1) * gw].double().cpu().numpy()
        got = o[gi * gw:(gi + 1) * gw].double().cpu().numpy()
        ref = O.oracle_divergence(d, p, n_e, g, U, PAR.nu, PAR.zeta, PAR.T, (1.0, 1.0, 1.0), with_source)
        real = np.broadcast_to((np.arange(g) < n_e)[None, None, :], (nv, npt, g)).reshape(-1)
        assert np.all(got[~real] == SENTINEL), f"group {gi}: kernel wrote into padding"
        maxdiff = max(maxdiff, float(np.max(np.abs(got - ref)[real])))
        maxref = max(maxref, float(np.max(np.abs(ref)[real])))
    err = maxdiff / max(1.0, maxref)
    tol = 1e-5 if fp32 else 1e-12
    assert err <= tol, f"d{d} p{p} n={n_elem} fp32={fp32} src={with_source}: rel err {err:.3e} over " \
                       f"{len(pick)} groups (last byte {words * wb})"
    del u, o
    torch.cuda.empty_cache()
    return err, len(pick), words * wb


@pytest.mark.parametrize("p,n_elem", [(3, 2343750), (5, 694445)])
def test_config5_full_field_sampled(cuda, p, n_elem):
    """BASELINE config 5: d=3 FP64, 1.5e8 solution points (15.6 GB per field)."""
    err, groups, nbytes = _sampled_parity(3, p, n_elem, False, False, 32, 500 + p)
    assert nbytes > 2 ** 32 and groups >= 32


def test_config5_p3_with_source(cuda):
    _sampled_parity(3, 3, 2343750, False, True, 16, 77)


@pytest.mark.parametrize("fp32", [True, False])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_config2_full_size_sampled(cuda, p, fp32):
    """BASELINE config 2: d=3, ~1e7 points per (p, precision)."""
    n = int(round(1e7 / (p + 1) ** 3))
    _sampled_parity(3, p, n, fp32, p % 2 == 0, 32, 900 + p)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_config3_full_size_sampled(cuda, p):
    """BASELINE config 3: d=2 FP32, 1e6 elements per order."""
    _sampled_parity(2, p, 1000000, True, p % 2 == 1, 32, 300 + p)


def test_bench_group_table_matches_library(cuda):
    """bench.py's static GPU_GROUPS (used by the reference arm, which must not load the
    B200 library) equals hf_preferred_group for every workload case."""
    import bench
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Precision
    for (d, p, prec), g in bench.GPU_GROUPS.items():
        assert hf.preferred_group(hf.make_problem(d, p, 1, 1, Precision[prec], PAR)) == g, (d, p, prec)
