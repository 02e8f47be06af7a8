"""Config-1-sized A/B (d3 p3 FP64, 32768 elements): lines variants back to back, 50 launches
between one event pair, round-robin over the candidates, 10 rounds; median fraction of the
roofline.  Tuning build.

    HEXFUSE_B200_LIB=.../lib_tuning/libhexfuse_b200.so python tools/small_ab.py 25 26 7
"""
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
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    d, p, prec, n = 3, 3, Precision.fp64, 32768
    variants = [int(v) for v in sys.argv[1:]] or [25, 26]
    npt = (p + 1) ** d
    u = torch.empty(n * npt * 13, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    o = torch.empty_like(u)
    alg = n * npt * 2 * 13 * 8
    runs = []
    for v in variants:
        g = hf.variant_info(hf.make_problem(d, p, 1, 1, prec, PAR), Method.lines, v)["elems_per_cta"]
        pr = hf.make_problem(d, p, n, g, prec, PAR)
        runs.append((v, hf.variant_info(pr, Method.lines, v)["name"],
                     (lambda pr=pr, v=v: hf.fused_divergence_variant(pr, Method.lines, v, u, o)), []))
    for _, _, fn, _ in runs:
        for _ in range(20):
            fn()
    torch.cuda.synchronize()
    for _ in range(10):
        for v, name, fn, ts in runs:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(50):
                fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3 / 50)
    for v, name, fn, ts in runs:
        t = statistics.median(ts)
        print(json.dumps({"variant": v, "kernel": name, "us": round(t * 1e6, 2), "frac": round(alg / t / 1e9 / peak, 4)}))


if __name__ == "__main__":
    main()
