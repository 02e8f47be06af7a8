"""Host-buffer path (hf_fused_divergence_host) against the PCIe ceiling, by base slice size:
config-1 and config-2-sized FP64 fields on pinned buffers, wall time per call (median of 7).
The slice size is read once per process (HF_HOST_SLICE_MB), so each size runs in a child.

    python tools/host_probe.py > profiles/r02/host_probe.jsonl
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, time, statistics, torch
sys.path.insert(0, ROOT)
import paper_2107_14027_b200 as hf
from paper_2107_14027_b200 import PhysParams, Precision
par = PhysParams(1 / 1600, 2.5, 1.0)
out = []
for d, p, n_pts in ((3, 3, 2097152), (3, 3, 1e7), (3, 6, 1e7)):
    prec = Precision.fp64
    g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, par))
    npt = (p + 1) ** d
    n = int(n_pts / npt) // g * g
    pr = hf.make_problem(d, p, n, g, prec, par)
    w = hf.field_words(pr)
    hu = torch.empty(w, dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
    ho = torch.empty_like(hu, pin_memory=True)
    ctx = hf.Context(0)
    ctx.run_batch([(pr, hu, ho)])
    ts = []
    for _ in range(7):
        t = time.perf_counter(); ctx.run_batch([(pr, hu, ho)]); ts.append(time.perf_counter() - t)
    ctx.close()
    t = statistics.median(ts)
    out.append({"slice_mb": int(os.environ.get("HF_HOST_SLICE_MB", "48")), "d": d, "p": p, "points": n * npt,
                "bytes_each_way": w * 8, "ms": round(t * 1e3, 3), "gdofs": round(n * npt / t / 1e9, 4),
                "GBps_each_way": round(w * 8 / t / 1e9, 2)})
print(json.dumps(out))
'''


def main():
    for mb in (8, 16, 24, 32, 48, 64, 96):
        env = dict(os.environ, HF_HOST_SLICE_MB=str(mb))
        r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + CHILD], env=env, capture_output=True, text=True)
        if r.returncode:
            print(json.dumps({"slice_mb": mb, "error": r.stderr[-400:]}), flush=True)
            continue
        for row in json.loads(r.stdout.strip().splitlines()[-1]):
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
