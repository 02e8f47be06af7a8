"""Worst field_rel_error (verify.hpp:19-33) of the selected kernel against the CPU
oracle per (d, p, precision), over random fields (3 seeds, +-source) and the TGV
fixture -- the margin to the north-star tolerances (1e-5 FP32, 1e-12 FP64).

    python tools/parity_errors.py [--out gpurun_out/parity_errors.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402  (test infrastructure: the checker)
import paper_2107_14027_b200 as hf  # noqa: E402
from gpu_util import PAR, run_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = []
    for d, pmax in ((3, 7), (2, 8)):
        for p in range(1, pmax + 1):
            for fp32 in (True, False):
                g = hf.preferred_group(hf.make_problem(d, p, 1, 1, int(not fp32), PAR))
                n = max(4 * g, (2000 // (p + 1) ** d) // g * g + 1)
                worst = 0.0
                for t in range(3):
                    U = O.random_field(d, p, n, g, fp32, 7000 + t)
                    for src in (False, True):
                        got = run_device(d, p, n, g, fp32, U, with_source=src)
                        ref = O.oracle_divergence(d, p, n, g, U, PAR.nu, PAR.zeta, PAR.T, (1.0, 1.0, 1.0), src)
                        worst = max(worst, O.field_rel_error(d, p, n, g, got, ref))
                if d == 3:
                    U = O.tgv_field(p, 64, g, fp32)
                    got = run_device(d, p, 64, g, fp32, U)
                    ref = O.oracle_divergence(d, p, 64, g, U, PAR.nu, PAR.zeta, PAR.T)
                    worst = max(worst, O.field_rel_error(d, p, 64, g, got, ref))
                tol = 1e-5 if fp32 else 1e-12
                row = {"d": d, "p": p, "precision": "fp32" if fp32 else "fp64",
                       "kernel": hf.kernel_info(hf.make_problem(d, p, n, g, int(not fp32), PAR))["name"],
                       "worst_rel_error": worst, "tolerance": tol, "margin": tol / max(worst, 1e-300)}
                print(json.dumps(row), flush=True)
                res.append(row)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
