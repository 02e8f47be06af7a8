"""Tile mode (hf_lines.cuh): time every one-chunk lines variant (NE0, NE0/2, NE0/4, 2 NE0)
on a caller-chosen AoSoA group, forced past the host's choice, to calibrate
lines_variant_for_group (hf_capi.cu).  ~1e7 points, median of 15 CUDA-event launches.

    python tools/tile_probe.py --d 3 --groups 8,12,16,20,24,32,40,64 > profiles/r02/tile_probe.jsonl
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--ps", default="")
    ap.add_argument("--groups", default="8,12,16,20,24,32,40,64")
    ap.add_argument("--points", type=float, default=1e7)
    ap.add_argument("--variants", default="7,1,0,2", help="lines variants to force (19-22: component split)")
    ap.add_argument("--precisions", default="fp32,fp64")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    ps = [int(x) for x in a.ps.split(",")] if a.ps else (list(range(1, 7)) if a.d == 3 else list(range(1, 9)))
    for prec in [Precision[x] for x in a.precisions.split(",")]:
        for p in ps:
            npt = (p + 1) ** a.d
            for g in [int(x) for x in a.groups.split(",")]:
                n = max(g, int(a.points / npt) // g * g)
                pr = hf.make_problem(a.d, p, n, g, prec, PAR)
                dt = torch.float32 if prec == Precision.fp32 else torch.float64
                u = torch.empty(hf.field_words(pr), dtype=dt, device="cuda").uniform_(-1, 1)
                o = torch.empty_like(u)
                auto = hf.kernel_info(pr)["name"]
                for v in [int(x) for x in a.variants.split(",")]:
                    try:
                        info = hf.variant_info(pr, Method.lines, v)
                        for _ in range(2):
                            hf.fused_divergence_variant(pr, Method.lines, v, u, o)
                    except Exception:
                        continue
                    ts = []
                    for _ in range(15):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        hf.fused_divergence_variant(pr, Method.lines, v, u, o)
                        e1.record()
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e-3)
                    t = statistics.median(ts)
                    ach = n * npt * 2 * hf.n_vars(a.d) * u.element_size() / t / 1e9
                    print(json.dumps({"d": a.d, "p": p, "precision": prec.name, "group": g, "variant": v,
                                      "ne": info["elems_per_cta"], "kernel": info["name"], "auto": auto,
                                      "blocks_per_sm": info["blocks_per_sm"], "us": round(t * 1e6, 2),
                                      "frac": round(ach / peak, 4)}), flush=True)
                del u, o
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
