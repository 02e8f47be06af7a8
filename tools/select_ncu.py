"""ncu counters for the method selection (tools/select_methods.py), per candidate kernel:
DRAM bytes read / written against the algorithmic bytes, and shared-memory bank
conflicts (l1tex__data_bank_conflicts_pipe_lsu_mem_shared) against the shared
wavefronts -- the planar kernels' padded plane buffer included.

Two steps on the GPU box (one ncu process over every candidate):

    ncu --metrics $(python tools/select_ncu.py --metrics) --clock-control none --csv \
        --log-file gpurun_out/sel_ncu.csv python tools/select_ncu.py --launch gpurun_out/sel_launches.json
    python tools/select_ncu.py --parse gpurun_out/sel_ncu.csv gpurun_out/sel_launches.json > profiles/.../sel_ncu.jsonl

--launch runs every candidate (method, variant) of every (d, p, precision) once on a
~2e6-point field (the counters are per-launch totals; their ratios to the algorithmic
bytes do not depend on the size) and records the launch order; --parse joins the ncu
rows to the candidates by that order.
"""
import argparse
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]


def launch(out_path, points, dims, variants):
    import torch

    from bench import launches_per_call

    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Method, PhysParams, Precision
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    order = []
    for d in dims:
        for prec in (Precision.fp32, Precision.fp64):
            for p in range(1, (7 if d == 3 else 8) + 1):
                cands = [(Method.lines, v) for v in variants]
                if d == 3:
                    cands += [(Method.planar, 0), (Method.planar_managed, 0)]
                npt = (p + 1) ** d
                n = max(512, int(points / npt) // 512 * 512)
                dt = torch.float32 if prec == Precision.fp32 else torch.float64
                words = n * npt * hf.n_vars(d)
                u = torch.rand(words, dtype=dt, device="cuda") * 2 - 1
                o = torch.empty_like(u)
                for meth, v in cands:
                    pr0 = hf.make_problem(d, p, 1, 1, prec, par, method=meth)
                    try:
                        info = hf.variant_info(pr0, meth, v)
                    except (hf.HexfuseInvalid, hf.HexfuseError):
                        continue
                    g = info["elems_per_cta"]
                    pr = hf.make_problem(d, p, n, g, prec, par, method=meth)
                    info = hf.variant_info(pr, meth, v)
                    hf.fused_divergence_variant(pr, meth, v, u, o)
                    torch.cuda.synchronize()
                    order.append({"d": d, "p": p, "precision": prec.name, "method": meth.name, "variant": v,
                                  "kernel": info["name"], "group": g, "n_elem": n, "points": n * npt,
                                  "alg_bytes": n * npt * 2 * hf.n_vars(d) * u.element_size(),
                                  "launches": launches_per_call(info, n, g, u.element_size(), words)})
                del u, o
                torch.cuda.empty_cache()
    with open(out_path, "w") as f:
        json.dump(order, f)


def parse(csv_path, order_path):
    txt = open(csv_path).read()
    txt = txt[txt.index('"ID"'):]
    per = {}
    for r in csv.DictReader(io.StringIO(txt)):
        if "hf_" not in r["Kernel Name"]:
            continue
        e = per.setdefault(int(r["ID"]), {"ncu_kernel": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] not in ("", "n/a") else None
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "usecond": 1e3, "us": 1e3,
                 "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        e[r["Metric Name"]] = v * scale if v is not None else None
    launches = [per[k] for k in sorted(per)]
    order = json.load(open(order_path))
    i = 0
    for c in order:
        ks = launches[i:i + c["launches"]]  # a TMA-ring call with a partial chunk launches a tail kernel too
        i += c["launches"]
        rd = sum(k.get("dram__bytes_read.sum") or 0 for k in ks)
        wr = sum(k.get("dram__bytes_write.sum") or 0 for k in ks)
        bc = sum(k.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") or 0 for k in ks)
        wf = sum(k.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or 0 for k in ks)
        ns = sum(k.get("gpu__time_duration.sum") or 0 for k in ks)
        c.update({"ncu_kernel": ks[0]["ncu_kernel"][:120], "ncu_ns": ns, "dram_read": rd, "dram_write": wr,
                  "traffic_alg_ratio": round((rd + wr) / c["alg_bytes"], 4),
                  # ncu flushes the caches before the launch, so reads are all DRAM; writes of a field
                  # smaller than L2 can still be dirty in L2 at kernel end -- the read ratio is the clean one
                  "read_alg_ratio": round(rd / (c["alg_bytes"] / 2), 4),
                  "bank_conflicts": bc, "shared_wavefronts": wf,
                  "conflict_per_wavefront": round(bc / wf, 4) if wf else None,
                  "bank_conflicts_ld": sum(k.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum") or 0
                                           for k in ks),
                  "bank_conflicts_st": sum(k.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum") or 0
                                           for k in ks)})
        print(json.dumps(c))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--metrics", action="store_true", help="print the metric list for ncu --metrics")
    ap.add_argument("--launch", default=None)
    ap.add_argument("--parse", nargs=2, default=None)
    ap.add_argument("--points", type=float, default=2e6)
    ap.add_argument("--dims", default="3,2")
    ap.add_argument("--variants", default=",".join(str(v) for v in range(28)))
    a = ap.parse_args()
    if a.metrics:
        print(",".join(METRICS))
    elif a.launch:
        launch(a.launch, a.points, [int(x) for x in a.dims.split(",")], [int(x) for x in a.variants.split(",")])
    elif a.parse:
        parse(*a.parse)


if __name__ == "__main__":
    main()
