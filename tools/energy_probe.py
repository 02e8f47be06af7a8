"""Energy per launch of candidate lines variants (NVML total-energy counter): each candidate
runs back to back for ~1.5 s on the same ~1e7-point field; reported are joules per launch,
nJ per algorithmic byte, the achieved fraction of the roofline and the median SM clock.
Under a power cap the SM clock follows the power draw, so at equal speed the variant that
spends fewer joules per byte keeps its clocks.  Tuning build (every variant):

    HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so \\
        python tools/energy_probe.py [--sweep profiles/r02/select/select_r02c.jsonl --top 5] > out.jsonl
"""
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml as N  # noqa: E402
import torch  # noqa: E402

import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)
CASES = [(3, 3, "fp64", [25, 26, 27, 7, 11, 19]), (3, 3, "fp32", [25, 26, 27, 7, 13]),
         (3, 5, "fp64", [1, 0, 20, 3]), (3, 6, "fp64", [3, 0, 1, 5]), (3, 4, "fp64", [20, 27, 7, 11])]


def cases_from_sweep(path, top, table):
    """Per (d, p, precision): the `top` fastest lines variants of a selection sweep, plus the
    selection table's current variant."""
    rows = [json.loads(x) for x in open(path) if x.strip()]
    out = []
    for key in sorted({(r["d"], r["p"], r["precision"]) for r in rows}):
        c = sorted([r for r in rows if (r["d"], r["p"], r["precision"]) == key and r["method"] == "lines"],
                   key=lambda r: -r["alg_GBps"])
        vs = [r["variant"] for r in c[:top]]
        cur = table.get(key)
        if cur is not None and cur not in vs:
            vs.append(cur)
        out.append((key[0], key[1], key[2], vs))
    return out


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", default=None, help="take the candidates from a select_methods.py sweep")
    ap.add_argument("--top", type=int, default=5)
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--rr", type=int, default=0,
                    help="round-robin: this many rounds of --seconds per candidate, candidates alternating "
                         "(drift in power and clocks hits every candidate alike); medians reported")
    ap.add_argument("--only", default=None, help="d:p:precision:v1/v2/... entries separated by ','")
    a = ap.parse_args()
    cases = CASES
    if a.sweep:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from select_methods import current_table
        cases = cases_from_sweep(a.sweep, a.top, current_table())
    if a.only:
        cases = []
        for ent in a.only.split(","):
            d, p, precn, vs = ent.split(":")
            cases.append((int(d), int(p), precn, [int(v) for v in vs.split("/")]))
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(0)
    if a.rr:
        return round_robin(h, cases, a)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for d, p, precn, variants in cases:
        prec = Precision[precn]
        npt = (p + 1) ** d
        n = int(1e7 / npt) // 512 * 512
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        u = torch.empty(n * npt * hf.n_vars(d), dtype=dt, device="cuda").uniform_(-1, 1)
        o = torch.empty_like(u)
        alg = n * npt * 2 * hf.n_vars(d) * u.element_size()
        for v in variants:
            pr0 = hf.make_problem(d, p, 1, 1, prec, PAR)
            try:
                g = hf.variant_info(pr0, Method.lines, v)["elems_per_cta"]
            except (hf.HexfuseInvalid, hf.HexfuseError):
                continue
            pr = hf.make_problem(d, p, n, g, prec, PAR)
            name = hf.variant_info(pr, Method.lines, v)["name"]
            for _ in range(20):
                hf.fused_divergence_variant(pr, Method.lines, v, u, o)
            torch.cuda.synchronize()
            clocks, stop = [], threading.Event()

            def sample():
                while not stop.is_set():
                    clocks.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    time.sleep(0.01)
            th = threading.Thread(target=sample, daemon=True)
            e0 = N.nvmlDeviceGetTotalEnergyConsumption(h)
            t0 = time.perf_counter()
            th.start()
            launches = 0
            while time.perf_counter() - t0 < a.seconds:
                for _ in range(50):
                    hf.fused_divergence_variant(pr, Method.lines, v, u, o)
                launches += 50
                torch.cuda.synchronize()
            t = time.perf_counter() - t0
            e1 = N.nvmlDeviceGetTotalEnergyConsumption(h)
            stop.set()
            th.join()
            joules = (e1 - e0) * 1e-3
            print(json.dumps({"d": d, "p": p, "precision": precn, "variant": v, "kernel": name,
                              "J_per_launch": round(joules / launches, 5),
                              "nJ_per_byte": round(joules / launches / alg * 1e9, 4),
                              "watts": round(joules / t, 1), "frac": round(alg * launches / t / 1e9 / peak, 4),
                              "sm_mhz_median": statistics.median(clocks) if clocks else None}), flush=True)
        del u, o
        torch.cuda.empty_cache()


def run_for(h, fn, seconds):
    """fn back to back for `seconds`: (launches, joules, seconds, median SM clock)."""
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            time.sleep(0.01)
    th = threading.Thread(target=sample, daemon=True)
    torch.cuda.synchronize()
    e0 = N.nvmlDeviceGetTotalEnergyConsumption(h)
    t0 = time.perf_counter()
    th.start()
    launches = 0
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            fn()
        launches += 20
        torch.cuda.synchronize()
    t = time.perf_counter() - t0
    e1 = N.nvmlDeviceGetTotalEnergyConsumption(h)
    stop.set()
    th.join()
    return launches, (e1 - e0) * 1e-3, t, (statistics.median(clocks) if clocks else None)


def round_robin(h, cases, a):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for d, p, precn, variants in cases:
        prec = Precision[precn]
        npt = (p + 1) ** d
        n = int(1e7 / npt) // 512 * 512
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        u = torch.empty(n * npt * hf.n_vars(d), dtype=dt, device="cuda").uniform_(-1, 1)
        o = torch.empty_like(u)
        alg = n * npt * 2 * hf.n_vars(d) * u.element_size()
        runs = []
        for v in variants:
            try:
                g = hf.variant_info(hf.make_problem(d, p, 1, 1, prec, PAR), Method.lines, v)["elems_per_cta"]
            except (hf.HexfuseInvalid, hf.HexfuseError):
                continue  # not instantiated (e.g. its shared memory exceeds a CTA)
            pr = hf.make_problem(d, p, n, g, prec, PAR)
            runs.append((v, hf.variant_info(pr, Method.lines, v)["name"],
                         (lambda pr=pr, v=v: hf.fused_divergence_variant(pr, Method.lines, v, u, o)), []))
        for _, _, fn, _ in runs:
            for _ in range(10):
                fn()
        for _ in range(a.rr):
            for v, name, fn, res in runs:
                res.append(run_for(h, fn, a.seconds))
        for v, name, fn, res in runs:
            fr = [alg * L / t / 1e9 / peak for L, J, t, mhz in res]
            nj = [J / L / alg * 1e9 for L, J, t, mhz in res]
            print(json.dumps({"d": d, "p": p, "precision": precn, "variant": v, "kernel": name,
                              "frac_median": round(statistics.median(fr), 4), "frac_all": [round(x, 4) for x in fr],
                              "nJ_per_byte_median": round(statistics.median(nj), 4),
                              "sm_mhz_median": statistics.median([m for *_, m in res if m])}), flush=True)
        del u, o
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
