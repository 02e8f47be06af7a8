"""Caller groups under sustained load: for the AoSoA groups the reference's presets produce
(presets.hpp:25-37, lines block / m^2) every one-chunk chunk size forced on the caller's group
(tile mode), candidates alternating in 0.4 s back-to-back slices, three rounds; the AUTO
choice (hf_capi.cu lines_variant_for_group) is marked.

    python tools/group_sustained.py > profiles/r02/groups_sustained/after.jsonl
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)
# (d, p, precision, caller group): the reference's preset groups and the lines defaults
CASES = [(3, 1, "fp32", 64), (3, 2, "fp32", 40), (3, 3, "fp32", 32), (3, 4, "fp32", 8),
         (3, 1, "fp64", 64), (3, 2, "fp64", 40), (3, 3, "fp64", 12), (3, 4, "fp64", 8),
         (3, 5, "fp64", 4), (3, 6, "fp64", 2), (3, 5, "fp32", 16), (3, 3, "fp64", 32)]


def slice_time(fn, seconds):
    torch.cuda.synchronize()
    t0, n = time.perf_counter(), 0
    while time.perf_counter() - t0 < seconds:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for d, p, precn, G in CASES:
        prec = Precision[precn]
        npt = (p + 1) ** d
        n = int(1e7 / npt) // G * G
        pr = hf.make_problem(d, p, n, G, prec, PAR)
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        u = torch.empty(hf.field_words(pr), dtype=dt, device="cuda").uniform_(-1, 1)
        o = torch.empty_like(u)
        alg = n * npt * 2 * hf.n_vars(d) * u.element_size()
        auto = hf.kernel_info(pr)["name"]
        runs = [("auto", auto, lambda: hf.fused_divergence_device(pr, u, o), [])]
        for v in (0, 1, 7, 2, 24):
            try:
                name = hf.variant_info(pr, Method.lines, v)["name"]
            except (hf.HexfuseInvalid, hf.HexfuseError):
                continue
            runs.append((v, name, (lambda v=v: hf.fused_divergence_variant(pr, Method.lines, v, u, o)), []))
        for _, _, fn, _ in runs:
            for _ in range(5):
                fn()
        for _ in range(3):
            for _, _, fn, ts in runs:
                ts.append(slice_time(fn, 0.4))
        for v, name, _, ts in runs:
            t = statistics.median(ts)
            print(json.dumps({"d": d, "p": p, "precision": precn, "group": G, "variant": v, "kernel": name,
                              "frac": round(alg / t / 1e9 / peak, 4)}), flush=True)
        del u, o
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
