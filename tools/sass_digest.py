"""SASS digest of the kernels the library selects (no GPU needed): for every (d, p,
precision) of the selection table, plus the planar methods (a) at d = 3, the
instruction mix that proves the design (UBLKCP / UTMALDG / UTMASTG bulk and tensor
copies, SYNCS mbarrier operations, FFMA2 / DFMA contraction, LDS / STS), registers,
local-memory (spill) bytes and static shared memory, from cuobjdump on the built
library.

    python tools/sass_digest.py [--lib paper_2107_14027_b200/lib/libhexfuse_b200.so] \
        --json profiles/r02/sass_digest.json --md profiles/r02/sass_digest.md
"""
import argparse
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

OPS = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "FFMA2", "FMUL2", "FADD2", "FFMA", "DFMA", "DMUL", "DADD", "LDS",
       "STS", "LDG", "STG", "BAR", "CALL"]


def resources(lib):
    out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        if name and "REG:" in line:
            res[name] = {k.lower(): int(v) for k, v in re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", line)}
            name = None
    return res


def mangled(info, d, p, prec, src=False):
    """The mangled name of the kernel that kernel_info describes (templates in hf_lines.cuh,
    hf_lines_pipe.cuh, hf_planar.cuh)."""
    R = "f" if prec == Precision.fp32 else "d"
    m = p + 1
    name = info["name"]
    ne = info["elems_per_cta"]
    b = "1" if src else "0"
    if name.startswith("hf_lines_pipe"):
        st = int(re.search(r"_s(\d+)", name).group(1))
        gr = re.search(r"_s\d+_g(\d+)", name)
        gr = int(gr.group(1)) if gr else 1
        cs = "1" if "_cs" in name else "0"
        tile = "1" if "_tile" in name else "0"  # variant 24 (the tile ring) is never a selected kernel
        return (f"_ZN3hfb20hf_lines_pipe_kernelI{R}Li{d}ELi{m}ELi{ne}ELi{st}ELi{gr}ELb{b}ELb0ELb{cs}ELb{tile}"
                "EEEvNS_6ParamsIT_EE")
    if name.startswith("hf_lines"):
        lpt = re.search(r"_l(\d+)", name)
        lpt = int(lpt.group(1)) if lpt else 1
        gs = re.search(r"_g(\d+)", name)
        gs = int(gs.group(1)) if gs else ne
        cs = "1" if "_cs" in name else "0"
        xp = 0
        if "_xp" in name:  # xpad_code (hf_lines.cuh): x-row pad words + 256 x k-plane pad rows
            w = 4 if prec == Precision.fp32 else 8
            if d == 3 and ne == 1 and (m * w) % 16 == 0:
                xp = 256
            else:
                gran = 16 // w
                while (m * ne + xp) % gran or ((m * ne + xp) // gran) % 2 == 0:
                    xp += 1
        return (f"_ZN3hfb15hf_lines_kernelI{R}Li{d}ELi{m}ELi{ne}ELb{b}ELi{lpt}ELb0ELi{gs}ELb{cs}ELi{xp}E"
                "EEvNS_6ParamsIT_EE")
    if name.startswith("hf_planar_managed"):
        return f"_ZN3hfb24hf_planar_managed_kernelI{R}Li{m}ELi{ne}ELb{b}EEEvNS_6ParamsIT_EE"
    if name.startswith("hf_planar"):
        return f"_ZN3hfb16hf_planar_kernelI{R}Li{m}ELi{ne}ELb{b}EEEvNS_6ParamsIT_EE"
    return None


def op_counts(lib, fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
    c = Counter()
    for line in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            c[m.group(1)] += 1
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2107_14027_b200", "lib", "libhexfuse_b200.so"))
    ap.add_argument("--json", default=None)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    res = resources(a.lib)
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    rows = []
    cases = []
    for d, pmax in ((3, 7), (2, 8)):
        for prec in (Precision.fp32, Precision.fp64):
            for p in range(1, pmax + 1):
                cases.append((d, p, prec, Method.auto))
    for prec in (Precision.fp32, Precision.fp64):
        for p in range(1, 8):
            cases.append((3, p, prec, Method.planar))
            cases.append((3, p, prec, Method.planar_managed))
    for d, p, prec, meth in cases:
        pr0 = hf.make_problem(d, p, 1, 1, prec, par, method=meth)
        g = hf.preferred_group(pr0)
        info = hf.kernel_info(hf.make_problem(d, p, 1000, g, prec, par, method=meth))
        fn = mangled(info, d, p, prec)
        if fn is None or fn not in res:
            rows.append({"d": d, "p": p, "precision": prec.name, "method": meth.name, "kernel": info["name"],
                         "mangled": fn, "found": False})
            continue
        c = op_counts(a.lib, fn)
        row = {"d": d, "p": p, "precision": prec.name, "method": meth.name, "kernel": info["name"], "found": True,
               "registers": res[fn]["reg"], "spill_local_bytes": res[fn]["local"], "stack": res[fn]["stack"],
               "static_shared": res[fn]["shared"], "dynamic_shared": info["shared_bytes"],
               "block": info["block_threads"], "sass_instructions": sum(c.values())}
        for op in OPS:
            row[op] = sum(v for k, v in c.items() if k == op or k.startswith(op + "."))
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)
    if a.md:
        with open(a.md, "w") as f:
            f.write("# SASS digest of the selected kernels (cuobjdump on the production library)\n\n"
                    "`tools/sass_digest.py`; the `auto` rows are the kernels the selection table runs for the "
                    "preferred group; `planar` / `planar_managed` are method (a).  Counts are static SASS "
                    "instructions (prefix match: `SYNCS` covers every `SYNCS.*`), registers and local-memory "
                    "(spill) bytes per thread from `cuobjdump -res-usage`.\n\n")
            cols = ["d", "p", "precision", "method", "kernel", "registers", "spill_local_bytes", "stack", "UBLKCP", "UTMALDG",
                    "UTMASTG", "SYNCS", "FFMA2", "FFMA", "DFMA", "LDS", "STS", "BAR", "sass_instructions"]
            f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
            for r in rows:
                f.write("| " + " | ".join(str(r.get(k, "")) for k in cols) + " |\n")
    missing = [r for r in rows if not r["found"]]
    if missing:
        print("not found:", [(r["kernel"], r["mangled"]) for r in missing], file=sys.stderr)


if __name__ == "__main__":
    main()
