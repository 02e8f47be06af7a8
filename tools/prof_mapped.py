"""Launch the mapped-element kernel (hf_mapped.cuh) for one (d, p, precision) a few times:
the command to put under `ncu --set full`.

    python tools/prof_mapped.py --d 3 --p 3 --prec fp64 --launches 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--prec", default="fp64")
    ap.add_argument("--points", type=float, default=1e7)
    ap.add_argument("--launches", type=int, default=2)
    a = ap.parse_args()
    prec = Precision[a.prec]
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    g = hf.mapped_kernel_info(hf.make_problem(a.d, a.p, 1, 1, prec, par))["elems_per_cta"]
    npt = (a.p + 1) ** a.d
    n = max(g, int(a.points / npt) // g * g)
    pr = hf.make_problem(a.d, a.p, n, g, prec, par)
    dt = torch.float32 if prec == Precision.fp32 else torch.float64
    u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda") * 2 - 1
    o = torch.empty_like(u)
    nc = 1 << a.d
    geo = torch.empty(hf.geometry_words(pr), dtype=dt, device="cuda")
    gv = geo.view(-1, nc, a.d, g)
    sign = torch.tensor([[1.0 if (c >> x) & 1 else -1.0 for x in range(a.d)] for c in range(nc)], dtype=dt,
                        device="cuda")
    gv.copy_((0.5 * sign)[None, :, :, None] + 0.075 * (torch.rand_like(gv) * 2 - 1))
    for _ in range(a.launches):
        hf.fused_divergence_mapped_device(pr, u, geo, o)
    torch.cuda.synchronize()
    print(hf.mapped_kernel_info(pr), n, "elements")


if __name__ == "__main__":
    main()
