"""Variant choice against problem size: every lines variant of a few (d, p, precision) at
sizes from 2e5 to 1e7 points, timed back to back (20 launches between one CUDA-event pair,
so consecutive launches overlap through programmatic dependent launch as in bench.py's timed
region).  Run against the tuning build, which carries every variant:

    HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so \\
        python tools/size_probe.py > profiles/r02/size_probe.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    cases = [(3, 3, Precision.fp64), (3, 5, Precision.fp64), (3, 1, Precision.fp32), (2, 1, Precision.fp32),
             (2, 2, Precision.fp32)]
    for d, p, prec in cases:
        npt = (p + 1) ** d
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        for pts in (2e5, 5e5, 1e6, 2.097152e6, 4e6, 1e7):
            n = max(512, int(pts / npt) // 512 * 512)
            words = n * npt * hf.n_vars(d)
            u = torch.empty(words, dtype=dt, device="cuda").uniform_(-1, 1)
            o = torch.empty_like(u)
            alg = n * npt * 2 * hf.n_vars(d) * u.element_size()
            rows = []
            for v in range(28):
                pr0 = hf.make_problem(d, p, 1, 1, prec, PAR)
                try:
                    info = hf.variant_info(pr0, Method.lines, v)
                except (hf.HexfuseInvalid, hf.HexfuseError):
                    continue
                g = info["elems_per_cta"]
                if n % g:
                    continue
                pr = hf.make_problem(d, p, n, g, prec, PAR)
                fn = (lambda pr=pr, v=v: hf.fused_divergence_variant(pr, Method.lines, v, u, o))
                for _ in range(5):
                    fn()
                torch.cuda.synchronize()
                best = None
                for _ in range(5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(20):
                        fn()
                    b.record()
                    b.synchronize()
                    t = a.elapsed_time(b) * 1e-3 / 20
                    best = t if best is None else min(best, t)
                rows.append((best, v, hf.variant_info(pr, Method.lines, v)["name"]))
            rows.sort()
            auto = hf.kernel_info(hf.make_problem(d, p, n, hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, PAR)),
                                                  prec, PAR))["name"]
            for t, v, name in rows[:6]:
                print(json.dumps({"d": d, "p": p, "precision": prec.name, "points": n * npt, "variant": v,
                                  "kernel": name, "us": round(t * 1e6, 2), "frac": round(alg / t / 1e9 / peak, 4),
                                  "auto_kernel": auto}), flush=True)
            del u, o
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
