"""Compare two tools/bench_fr.py sweeps (per (p, precision): correction and residual times)."""
import json
import sys

a = {(r["p"], r["precision"]): r for r in map(json.loads, open(sys.argv[1]))}
b = {(r["p"], r["precision"]): r for r in map(json.loads, open(sys.argv[2]))}
keys = sys.argv[3:] or ["fused_us", "project_us", "correct_us", "residual_us"]
for k in sorted(a):
    if k in b:
        print(k, "  ".join(f"{x} {a[k][x]:.0f}->{b[k][x]:.0f}" for x in keys))
