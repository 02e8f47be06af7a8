"""Small problems (BASELINE config 1: 2.1e6 points): where the fixed cost of a launch goes.
For a few (d, p, precision) and sizes from one chunk to 1e7 points, the selected kernel's
time (a) per launch between CUDA events and (b) per launch in a back-to-back run of 20
launches between one event pair (programmatic dependent launch can overlap consecutive
launches only there).  The intercept of time vs bytes is the fixed cost.

    python tools/small_probe.py > profiles/r02/small_probe.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    tag = os.environ.get("PROBE_TAG", "")
    for d, p, prec in ((3, 3, Precision.fp64), (3, 1, Precision.fp32), (2, 1, Precision.fp32), (3, 6, Precision.fp64)):
        g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR))
        npt = (p + 1) ** d
        for pts in (npt * g, 1e5, 5e5, 1e6, 2.097152e6, 4e6, 1e7):
            n = max(g, int(pts / npt) // g * g)
            pr = hf.make_problem(d, p, n, g, prec, PAR)
            dt = torch.float32 if prec == Precision.fp32 else torch.float64
            u = torch.empty(hf.field_words(pr), dtype=dt, device="cuda").uniform_(-1, 1)
            o = torch.empty_like(u)
            for _ in range(5):
                hf.fused_divergence_device(pr, u, o)
            torch.cuda.synchronize()
            ts = []
            for _ in range(30):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                hf.fused_divergence_device(pr, u, o)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e-3)
            t_ev = statistics.median(ts)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                hf.fused_divergence_device(pr, u, o)
            b.record()
            b.synchronize()
            t_bb = a.elapsed_time(b) * 1e-3 / 20
            byt = n * npt * 2 * hf.n_vars(d) * u.element_size()
            print(json.dumps({"tag": tag, "d": d, "p": p, "precision": prec.name, "kernel": hf.kernel_info(pr)["name"],
                              "n_elem": n, "points": n * npt, "bytes": byt, "us_event": round(t_ev * 1e6, 2),
                              "us_back_to_back": round(t_bb * 1e6, 2), "frac_event": round(byt / t_ev / 1e9 / peak, 4),
                              "frac_b2b": round(byt / t_bb / 1e9 / peak, 4)}), flush=True)
            del u, o


if __name__ == "__main__":
    main()
