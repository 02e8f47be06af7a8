"""Turn an ncu launch list of `bench.py` (gpu__time_duration + dram bytes per
launch) into profiles/ncu_traffic.json: per bench case, the DRAM bytes one
launch moved vs its algorithmic bytes, and the kernel's share of the step.

    python tools/ncu_traffic.py gpurun_out/launches.csv gpurun_out/bench.json profiles/ncu_traffic.json
"""
import csv
import io
import json
import sys
from collections import OrderedDict


def load_launches(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    per = OrderedDict()
    for r in csv.DictReader(io.StringIO(txt)):
        if "hf_" not in r["Kernel Name"]:
            continue
        e = per.setdefault(r["ID"], {"kernel": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            e["ns"] = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        else:
            e[r["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return list(per.values())


def main(csv_path, bench_path, out_path, steps=None):
    """`steps`: the leading step-major steps of the launch list to use (bench.py's warm-up
    steps; its roofline pass is case-major)."""
    launches = load_launches(csv_path)
    bench = json.loads(open(bench_path).read().strip().splitlines()[-1])
    cases = bench["cases"]
    n = len(cases)
    steps = int(steps) if steps else len(launches) // n
    out = {"source": {"launch_list": csv_path, "bench_line": bench_path,
                      "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                              "--clock-control none (cold-cache, serialised launches; compare shares, not "
                              "absolute times)"}}
    tot_ns = 0.0
    rows = []
    for i, c in enumerate(cases):
        ls = [launches[k * n + i] for k in range(steps)]
        rd = sum(x["dram__bytes_read.sum"] for x in ls) / steps
        wr = sum(x["dram__bytes_write.sum"] for x in ls) / steps
        ns = sum(x["ns"] for x in ls) / steps
        wb = 4 if c["precision"] == "fp32" else 8
        nv = 13 if c["d"] == 3 else 7
        alg = c["points"] * 2 * nv * wb
        rows.append((c["kernel"], {"ncu_kernel": ls[0]["kernel"], "dram_bytes_per_launch": rd + wr,
                                   "dram_read": rd, "dram_write": wr, "alg_bytes_per_launch": alg,
                                   "traffic_over_alg": (rd + wr) / alg, "ncu_us": ns / 1e3,
                                   "bench_us": c["us_per_launch"]}))
        tot_ns += ns
    tot_bench = sum(c["us_per_launch"] for c in cases)
    for (name, r), c in zip(rows, cases):
        r["ncu_share"] = r["ncu_us"] * 1e3 / tot_ns
        r["bench_share"] = c["us_per_launch"] / tot_bench
        out[name] = r
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    for name, r in rows:
        print(f"{name:40s} traffic/alg {r['traffic_over_alg']:.3f}  ncu share {r['ncu_share']:.3f}  "
              f"bench share {r['bench_share']:.3f}  ncu {r['ncu_us']:.1f} us  bench {r['bench_us']:.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:5])
