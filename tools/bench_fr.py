"""Time the FR stages around the fused kernel on a periodic mesh (~1e7 points):
fused divergence (stages 2+3+6), face projection (stage 1) and the interface
correction (stages 4+5), each with its algorithmic HBM bytes:

  fused    2 n_v m^d w per element
  project  n_v m^d w  read + F w written,      F = 2 d m^(d-1) n_v (face words per element)
  correct  F w read + 2 n_v m^d w (read-modify-write of the residual); every face array
           word is read twice (own side, neighbour side) but is unique data once, the
           second read an L2 hit when the neighbour's chunk is close in launch order
  residual (hf_fr_residual: the fused kernel writes the faces, then the correction)
           2 n_v m^d w + F w  +  F w + 2 n_v m^d w

    python tools/bench_fr.py [--points 1e7] [--dims 3,2] [--out gpurun_out/fr.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ts = []
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
    ap.add_argument("--out", default=None)
    ap.add_argument("--dims", default="3", help="comma list of dimensions (3, 2)")
    ap.add_argument("--sustained", type=float, default=0.0,
                    help="time each stage back to back for this many seconds (power-capped regime)")
    a = ap.parse_args()
    global timed
    if a.sustained > 0:
        def timed(fn, iters=0):  # noqa: F811 -- sustained mode
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            t0, n = time.perf_counter(), 0
            while time.perf_counter() - t0 < a.sustained:
                for _ in range(10):
                    fn()
                n += 10
                torch.cuda.synchronize()
            return (time.perf_counter() - t0) / n
    fh = open(a.out, "w") if a.out else None
    for d, prec, p in [(d, prec, p) for d in map(int, a.dims.split(",")) for prec in (Precision.fp32, Precision.fp64)
                       for p in range(1, 7 if d == 3 else 9)]:
        w = 4 if prec == Precision.fp32 else 8
        m = p + 1
        g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
        if d == 3:
            # periodic box nx x ny x nz with nx*ny a multiple of the group (layer partitions)
            nx = ny = max(2, round((a.points / m ** 3) ** (1 / 3)))
            while (nx * ny) % g:
                nx += 1
            nz = max(2, round(a.points / m ** 3 / (nx * ny)))
            dims = (nx, ny, nz)
        else:
            nx = max(2, round((a.points / m ** 2) ** 0.5))
            while nx % g:
                nx += 1
            dims = (nx, max(2, round(a.points / m ** 2 / nx)))
        n = int(np.prod(dims))
        pr = hf.make_problem(d, p, n, g, prec, PAR)
        dt = torch.float32 if w == 4 else torch.float64
        u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda") * 2 - 1
        out = torch.empty_like(u)
        uf = torch.empty(hf.face_words(pr), dtype=dt, device="cuda")
        ms = hf.make_mesh(dims, d)
        t_div = timed(lambda: hf.fused_divergence_device(pr, u, out))
        t_prj = timed(lambda: hf.fr_project_device(pr, u, uf))
        t_cor = timed(lambda: hf.fr_correct_device(pr, ms, uf, out))
        t_all = timed(lambda: hf.fr_residual_device(pr, dims, u, uf, out))
        nv, F = hf.n_vars(d), 2 * d * m ** (d - 1) * hf.n_vars(d)
        field = n * nv * m ** d * w
        faces = n * F * w
        row = {"d": d, "p": p, "precision": prec.name, "dims": dims, "points": n * m ** d,
               "fused_us": round(t_div * 1e6, 1), "fused_GBps": round(2 * field / t_div / 1e9, 1),
               "project_us": round(t_prj * 1e6, 1), "project_GBps": round((field + faces) / t_prj / 1e9, 1),
               "correct_us": round(t_cor * 1e6, 1), "correct_GBps": round((faces + 2 * field) / t_cor / 1e9, 1),
               "residual_us": round(t_all * 1e6, 1),
               "residual_gdofs": round(n * m ** d / t_all / 1e9, 3),
               "residual_GBps_alg": round((4 * field + 2 * faces) / t_all / 1e9, 1)}
        print(json.dumps(row), flush=True)
        if fh:
            fh.write(json.dumps(row) + "\n")
        del u, out, uf


if __name__ == "__main__":
    main()
