"""Launch one (d, p, precision, method, variant) configuration a few times -- a
short command to put under `ncu --set full` (one GPU, a handful of launches).

    python tools/prof_one.py --d 3 --p 6 --prec fp32 --variant 3 --points 1e7 --launches 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--prec", default="fp64")
    ap.add_argument("--method", default="lines")
    ap.add_argument("--variant", type=int, default=0, help="lines variant; -1 = the selected kernel (method auto)")
    ap.add_argument("--points", type=float, default=1e7)
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--src", action="store_true")
    ap.add_argument("--group", type=int, default=0, help="AoSoA group (default: the kernel's chunk)")
    a = ap.parse_args()
    prec = Precision[a.prec]
    method = Method[a.method]
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    pr0 = hf.make_problem(a.d, a.p, 1, 1, prec, par)
    if a.variant < 0:
        method = Method.auto
        g = hf.preferred_group(pr0)
    else:
        g = hf.variant_info(pr0, method, a.variant)["elems_per_cta"] if method != Method.unfused else 32
    if a.group > 0:
        g = a.group
    npt = (a.p + 1) ** a.d
    n = max(g, int(a.points / npt) // g * g)
    pr = hf.make_problem(a.d, a.p, n, g, prec, par, with_source=a.src, method=method)
    dt = torch.float32 if prec == Precision.fp32 else torch.float64
    u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda") * 2 - 1
    o = torch.empty_like(u)
    ws = None
    if method == Method.unfused:
        ws = torch.empty(hf.unfused_workspace_bytes(pr) // u.element_size(), dtype=dt, device="cuda")
    for _ in range(a.launches):
        if ws is not None:
            hf.unfused_divergence_device(pr, u, o, ws)
        elif a.variant < 0:
            hf.fused_divergence_device(pr, u, o)
        else:
            hf.fused_divergence_variant(pr, method, a.variant, u, o)
    torch.cuda.synchronize()
    print(hf.kernel_info(pr) if a.variant < 0 else
          (hf.variant_info(pr, method, a.variant) if ws is None else "unfused"), n, "elements")


if __name__ == "__main__":
    main()
