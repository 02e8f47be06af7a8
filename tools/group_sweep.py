"""Fused kernel throughput for caller-chosen AoSoA groups (tile mode, hf_lines.cuh).

For every (d, p, precision) of a workload and every group, the AUTO kernel on a
~1e7-point field (resident, > L2): median CUDA-event time of 20 launches, achieved
HBM GB/s on the algorithmic bytes (2 n_v w per point), fraction of the measured peak,
the kernel that ran, and the worst relative error of 4 sampled groups vs the oracle.

    python tools/group_sweep.py [--d 3] [--groups 1,8,12,...] > profiles/r02/groups.jsonl
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--ps", default="")
    ap.add_argument("--groups", default="")
    ap.add_argument("--points", type=float, default=1e7)
    ap.add_argument("--launches", type=int, default=20)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    ps = [int(x) for x in a.ps.split(",")] if a.ps else (list(range(1, 7)) if a.d == 3 else list(range(1, 9)))
    for prec in (Precision.fp32, Precision.fp64):
        for p in ps:
            m = p + 1
            pref = hf.preferred_group(hf.make_problem(a.d, p, 1, 1, prec, PAR))
            groups = [int(x) for x in a.groups.split(",")] if a.groups else \
                sorted({1, 8, 12, 15, 16, 20, 24, 32, 40, 64, 4 * (32 // m), pref})
            for g in groups:
                npt = m ** a.d
                n = max(g, int(a.points / npt) // g * g)
                pr = hf.make_problem(a.d, p, n, g, prec, PAR)
                dt = torch.float32 if prec == Precision.fp32 else torch.float64
                words = hf.field_words(pr)
                u = torch.empty(words, dtype=dt, device="cuda").uniform_(-1, 1)
                o = torch.empty_like(u)
                for _ in range(3):
                    hf.fused_divergence_device(pr, u, o)
                ts = []
                for _ in range(a.launches):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    hf.fused_divergence_device(pr, u, o)
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                t = statistics.median(ts)
                w = u.element_size()
                ach = n * npt * 2 * hf.n_vars(a.d) * w / t / 1e9
                # parity on 4 sampled groups (checker)
                nv = hf.n_vars(a.d)
                gw = g * npt * nv
                ng = -(-n // g)
                err = 0.0
                for gi in sorted({0, ng - 1, ng // 3, (2 * ng) // 3}):
                    U = u[gi * gw:(gi + 1) * gw].double().cpu().numpy()
                    got = o[gi * gw:(gi + 1) * gw].double().cpu().numpy()
                    ref = O.oracle_divergence(a.d, p, g, g, U, PAR.nu, PAR.zeta, PAR.T)
                    err = max(err, float(np.max(np.abs(got - ref))) / max(1.0, float(np.max(np.abs(ref)))))
                info = hf.kernel_info(pr)
                print(json.dumps({"d": a.d, "p": p, "precision": prec.name, "group": g, "preferred": pref,
                                  "n_elem": n, "kernel": info["name"], "us": round(t * 1e6, 2),
                                  "GBps": round(ach, 1), "frac": round(ach / peak, 4), "rel_err": float(f"{err:.3e}")}),
                      flush=True)
                del u, o
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
