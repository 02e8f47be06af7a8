"""Time the mapped-element kernel (non-constant Jacobian, hf_mapped.cuh) beside the
constant-Jacobian fused kernel on the same field: GDoF/s and achieved HBM GB/s
with algorithmic bytes = 2 n_v w per point + 2^d d w per element (geometry).

    python tools/bench_mapped.py [--points 1e7] [--dims 3,2] [--out gpurun_out/mapped.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=float, default=1e7)
    ap.add_argument("--dims", default="3,2")
    ap.add_argument("--out", default=None)
    ap.add_argument("--sustained", type=float, default=0.0,
                    help="time each case back to back for this many seconds (power-capped regime) instead of "
                         "the median of 20 event-bracketed launches")
    a = ap.parse_args()
    global timed
    if a.sustained > 0:
        def timed(fn, iters=0):  # noqa: F811 -- sustained mode
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
            t0, n = time.perf_counter(), 0
            while time.perf_counter() - t0 < a.sustained:
                for _ in range(20):
                    fn()
                n += 20
                torch.cuda.synchronize()
            return (time.perf_counter() - t0) / n
    fh = open(a.out, "w") if a.out else None
    for d in [int(x) for x in a.dims.split(",")]:
        for prec in (Precision.fp32, Precision.fp64):
            for p in range(1, (7 if d == 3 else 9)):
                w = 4 if prec == Precision.fp32 else 8
                info = hf.mapped_kernel_info(hf.make_problem(d, p, 1, 1, prec, PAR))
                g = info["elems_per_cta"]
                npt = (p + 1) ** d
                n = max(g, int(a.points / npt) // g * g)
                pr = hf.make_problem(d, p, n, g, prec, PAR)
                dt = torch.float32 if w == 4 else torch.float64
                u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda") * 2 - 1
                o = torch.empty_like(u)
                # boxes of half-width 0.5 with corners displaced by up to 15 %
                geo = torch.empty(hf.geometry_words(pr), dtype=dt, device="cuda")
                nc = 1 << d
                gv = geo.view(-1, nc, d, g)
                sign = torch.tensor([[1.0 if (c >> x) & 1 else -1.0 for x in range(d)] for c in range(nc)],
                                    dtype=dt, device="cuda")
                gv.copy_((0.5 * sign)[None, :, :, None] + 0.075 * (torch.rand_like(gv) * 2 - 1))
                t_map = timed(lambda: hf.fused_divergence_mapped_device(pr, u, geo, o))
                pr_c = hf.make_problem(d, p, n, hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR)), prec, PAR)
                t_con = None
                if hf.field_words(pr_c) == u.numel():
                    t_con = timed(lambda: hf.fused_divergence_device(pr_c, u, o))
                pts = n * npt
                alg = pts * 2 * hf.n_vars(d) * w + n * nc * d * w
                row = {"d": d, "p": p, "precision": prec.name, "kernel": info["name"], "n_elem": n, "points": pts,
                       "us": round(t_map * 1e6, 2), "gdofs": round(pts / t_map / 1e9, 3),
                       "alg_GBps": round(alg / t_map / 1e9, 1), "regs": hf.mapped_kernel_info(pr)["registers"],
                       "smem": info["shared_bytes"], "block": info["block_threads"],
                       "constant_jac_us": round(t_con * 1e6, 2) if t_con else None}
                print(json.dumps(row), flush=True)
                if fh:
                    fh.write(json.dumps(row) + "\n")
                del u, o, geo


if __name__ == "__main__":
    main()
