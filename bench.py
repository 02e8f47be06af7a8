"""Benchmark driver for the B200 fused flux + divergence kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config2|config1|config3|config4|config5]
                    [--impl ours|reference] [--scaling weak|strong] [--no-e2e]

Metric (BASELINE.json): GDoF/s = solution-point updates per second (all n_v
variables of a point = one update), with the fraction of the HBM roofline of
the dominant kernel (algorithmic bytes = n_v words read + n_v words written
per point, io_model Fused23, io_model.hpp:35).

Default workload = BASELINE config 2, the single-GPU case the metric is quoted
on: d=3 hexes, p = 1..6, FP32 and FP64, ~1e7 solution points per (p,
precision).  One step = one fused launch per (p, precision) = 12 launches over
resident synthetic inputs (uniform(-1,1), every case's input larger than L2).

Under torchrun (N > 1) each rank owns its own element slice (no data-path
collective; the NCCL group is only used for the barrier and the max-over-ranks
of the device time).  `value` is the whole-job aggregate.

`--impl reference` times the reference's own CPU implementation
(hexfuse::oracle_divergence compiled from /root/reference by oracle/Makefile
into oracle/_ref/libhexfuse_ref.so) on the host cores for a bounded sample of
the same workload; rank 0 alone runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024


# ------------------------------------------------------------------------------------------------ workloads
def workload_cases(name: str):
    """List of (d, p, precision_name, target_points) for a workload."""
    if name == "config2":
        return [(3, p, prec, 1e7) for prec in ("fp32", "fp64") for p in range(1, 7)]
    if name == "config1":
        return [(3, 3, "fp64", 32768 * 64)]
    if name == "config3":
        return [(2, p, "fp32", 1e6 * (p + 1) ** 2) for p in range(1, 9)]
    if name == "config4":
        return [(3, 4, "fp32", 1e7)]
    if name == "config5":
        return [(3, 3, "fp64", 1.5e8), (3, 5, "fp64", 1.5e8)]
    raise SystemExit(f"unknown workload {name}")


WORKLOAD_DESC = {
    "config2": "d3 hex order sweep p=1..6, fp32+fp64, ~1e7 points per case (BASELINE config 2)",
    "config1": "d3 hex p=3 fp64, 32768 elements (BASELINE config 1)",
    "config3": "d2 quad p=1..8 fp32, 1e6 elements per case (BASELINE config 3)",
    "config4": "d3 hex p=4 fp32, ~1e7 points, fused (BASELINE config 4; unfused timed beside it)",
    "config5": "d3 hex p=3 and p=5 fp64, 1.5e8 points (BASELINE config 5)",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    """Per-launch DRAM bytes of our kernels from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons through NVML every ~10 ms while running."""

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            self._ok = False
        self._t = threading.Thread(target=self._run, daemon=True)

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.N.nvmlDeviceGetClockInfo(self.h, self.N.NVML_CLOCK_SM))
                r = self.N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in self._NAMES.items():
                    if r & bit and nm != "gpu_idle":
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------ ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import Method, PhysParams, Precision

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    peak, peak_src = load_peaks()
    traffic = load_traffic()
    st = torch.cuda.current_stream()

    # ---- allocate every case's resident input/output on this rank
    cases = []
    gen = torch.Generator(device=dev)
    gen.manual_seed(2024 + rank)
    for (d, p, precn, target) in workload_cases(args.workload):
        prec = Precision[precn]
        g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, par))
        npt = (p + 1) ** d
        n_total = max(g, int(round(target / npt / g)) * g)
        if world > 1 and args.scaling == "strong":
            full = hf.make_problem(d, p, n_total, g, prec, par)
            _, n_elem, _ = hf.partition(full, world, rank)
        else:
            n_elem = n_total
        pr = hf.make_problem(d, p, n_elem, g, prec, par)
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        words = hf.field_words(pr)
        u = torch.empty(words, dtype=dt, device=dev)
        u.uniform_(-1.0, 1.0, generator=gen)
        o = torch.empty_like(u)
        wb = 4 if prec == Precision.fp32 else 8
        info = hf.kernel_info(pr)
        cases.append({"d": d, "p": p, "precision": precn, "pr": pr, "u": u, "o": o, "n_elem": n_elem,
                      "points": n_elem * npt, "alg_bytes": n_elem * npt * 2 * hf.n_vars(d) * wb,
                      "kernel": info["name"], "group": g, "info": info})
        assert u.numel() * wb * 2 > L2_BYTES or args.workload == "config3", "input must exceed L2"

    def step(record=None):
        for i, c in enumerate(cases):
            if record is not None:
                record[i][0].record(st)
            hf.fused_divergence_device(c["pr"], c["u"], c["o"], st)
            if record is not None:
                record[i][1].record(st)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-launch events + one pair around everything
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in cases]
          for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        t0.record(st)
        for k in range(args.steps):
            step(ev[k])
        t1.record(st)
        torch.cuda.synchronize()
        barrier()
    elapsed = t0.elapsed_time(t1) * 1e-3
    per_case = [[ev[k][i][0].elapsed_time(ev[k][i][1]) * 1e-3 for k in range(args.steps)] for i in range(len(cases))]
    if world > 1:
        tt = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    points_rank = sum(c["points"] for c in cases)
    points_all = points_rank * world if not (world > 1 and args.scaling == "strong") else None
    if points_all is None:
        pt = torch.tensor([float(points_rank)], device=dev, dtype=torch.float64)
        dist.all_reduce(pt, op=dist.ReduceOp.SUM)
        points_all = float(pt.item())
    value = points_all * args.steps / elapsed / 1e9

    # ---- per-case roofline, dominant kernel
    case_rows = []
    for c, ts in zip(cases, per_case):
        tavg = sum(ts) / len(ts)
        ach = c["alg_bytes"] / tavg / 1e9
        case_rows.append({"d": c["d"], "p": c["p"], "precision": c["precision"], "kernel": c["kernel"],
                          "n_elem": c["n_elem"], "group": c["group"], "points": c["points"],
                          "us_per_launch": round(tavg * 1e6, 2), "gdofs": round(c["points"] / tavg / 1e9, 3),
                          "achieved_GBps": round(ach, 1), "frac": round(ach / peak, 4),
                          "share_of_step": None})
    tot = sum(r["us_per_launch"] for r in case_rows)
    for r in case_rows:
        r["share_of_step"] = round(r["us_per_launch"] / tot, 4)
    dom = max(case_rows, key=lambda r: r["us_per_launch"])
    tr = traffic.get(dom["kernel"])
    roofline = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved_GBps"], "peak": peak,
                "unit": "GB/s", "frac": dom["frac"],
                "traffic": (tr["dram_bytes_per_launch"] if tr else None),
                "traffic_alg_ratio": (round(tr["dram_bytes_per_launch"] / tr["alg_bytes_per_launch"], 4)
                                      if tr else None),
                "peak_source": peak_src,
                "bytes_per_point": "2*n_v*w (n_v=13 d3 / 7 d2; w=4 fp32 / 8 fp64)"}
    agg_bytes = sum(c["alg_bytes"] for c in cases) * args.steps
    roofline["step_aggregate_frac"] = round(agg_bytes / elapsed / 1e9 / peak, 4)  # all launches of the step, per rank

    # ---- e2e through the host-buffer C ABI (pinned host buffers; H2D + kernel + D2H timed)
    e2e = None
    if not args.no_e2e:
        # Host memory: every rank pins an input and an output copy of its cases.  When
        # that would exceed a quarter of the host's RAM across the node's ranks, each
        # case is cut to a group-aligned prefix of its elements (elements are
        # independent, so GDoF/s is unchanged; the bytes per step are reported).
        host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        full_bytes = sum(2 * c["u"].numel() * c["u"].element_size() for c in cases)
        frac = min(1.0, 0.25 * host_ram / max(1, full_bytes * world))
        frac = min(frac, float(os.environ.get("HF_E2E_HOST_FRAC", "1")))  # test hook
        ctx = hf.Context(local_rank)
        hosts = []
        for c in cases:
            g = c["group"]
            n_e = c["n_elem"] if frac >= 1.0 else max(g, int(c["n_elem"] * frac) // g * g)
            pr_e = hf.make_problem(c["d"], c["p"], n_e, g, c["pr"].precision,
                                   PhysParams(c["pr"].nu, c["pr"].zeta, c["pr"].T))
            words = hf.field_words(pr_e)
            hu = torch.empty(words, dtype=c["u"].dtype, pin_memory=True)
            hu.copy_(c["u"][:words])
            ho = torch.empty_like(hu, pin_memory=True)
            hosts.append((hu, ho, pr_e, n_e * (c["p"] + 1) ** c["d"]))
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        # one step = every case of the workload through ONE copy pipeline
        # (hf_fused_divergence_host_batch: fill before the first case, drain after the last)
        batch = [(pr_e, hu, ho) for hu, ho, pr_e, _ in hosts]
        ctx.run_batch(batch)  # warm (allocates the context's slots)
        barrier()
        ta = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.run_batch(batch)
        tb = time.perf_counter()
        barrier()
        te = tb - ta
        if world > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        pts_e = sum(h[3] for h in hosts) * (world if not (world > 1 and args.scaling == "strong") else 1)
        if world > 1 and args.scaling == "strong":
            pt = torch.tensor([float(sum(h[3] for h in hosts))], device=dev, dtype=torch.float64)
            dist.all_reduce(pt, op=dist.ReduceOp.SUM)
            pts_e = float(pt.item())
        h2d = sum(h[0].numel() * h[0].element_size() for h in hosts)
        e2e = {"value": round(pts_e * e2e_steps / te / 1e9, 4), "unit": "GDoF/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d, "steps": e2e_steps,
               "path": "hf_fused_divergence_host_batch (pinned host buffers, one 3-stream slice pipeline per step)"}
        if frac < 1.0:
            e2e["sample"] = f"each case cut to {frac:.3f} of its elements (host RAM {host_ram / 2**30:.0f} GiB)"
        # the first e2e step's result must equal the device-resident run's result
        same = all(torch.equal(h[1].to(dev), c["o"][: h[1].numel()]) for h, c in zip(hosts, cases))
        e2e["matches_device_result"] = bool(same)
        ctx.close()
        del hosts

    # ---- unfused comparator beside it (config 4)
    unfused = None
    if args.workload == "config4":
        c = cases[0]
        ws = torch.empty(hf.unfused_workspace_bytes(c["pr"]) // c["u"].element_size(), dtype=c["u"].dtype,
                         device=dev)
        for _ in range(3):
            hf.unfused_divergence_device(c["pr"], c["u"], c["o"], ws, st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.steps):
            hf.unfused_divergence_device(c["pr"], c["u"], c["o"], ws, st)
        b.record(st)
        torch.cuda.synchronize()
        tu = a.elapsed_time(b) * 1e-3 / args.steps
        unfused = {"us_per_step": round(tu * 1e6, 2), "gdofs": round(c["points"] / tu / 1e9, 3),
                   "fused_speedup": round(tu / (case_rows[0]["us_per_launch"] * 1e-6), 3),
                   "model_speedup": 4.0}

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args, n_threads=args.cpu_threads)

    if rank == 0:
        line = {
            "metric": "GDoF/s (solution-point updates/sec), fused flux+divergence; roofline = fraction of HBM",
            "value": round(value, 4), "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps * 1e3, 4),
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32+f64" if args.workload in ("config2",) else
            ("f64" if all(c["precision"] == "fp64" for c in cases) else "f32"),
            "data": "synthetic uniform(-1,1) fields, resident in HBM",
            "config": {"workload": args.workload, "description": WORKLOAD_DESC[args.workload],
                       "cases": len(cases), "points_per_rank_per_step": points_rank,
                       "l2": "no flush; every case's input+output (>=0.4 GB) exceeds the 126 MB L2",
                       "method": "auto (measured selection table)", "parallelism": f"element-partition x{world}"},
            "roofline": roofline, "cases": case_rows, "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": args.steps * len(cases), "clocks": clk.summary(),
        }
        if unfused:
            line["unfused"] = unfused
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------ reference CPU
def cpu_sample_cases(args, budget_points):
    """Bounded, group-aligned sample of every case of the workload (same d, p, precision, group)."""
    import oracle as O  # noqa: F401  (test infrastructure: the CPU baseline leg only)
    from paper_2107_14027_b200 import PhysParams, Precision
    import paper_2107_14027_b200 as hf
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    out = []
    cases = workload_cases(args.workload)
    for (d, p, precn, target) in cases:
        prec = Precision[precn]
        g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, par))
        npt = (p + 1) ** d
        n = max(g, int(budget_points / len(cases) / npt) // g * g)
        out.append((d, p, precn, g, n))
    return out


def ref_supports(d, p):
    """The reference oracle's domain: gauss_legendre_points accepts m <= 8 (operators.hpp:18)."""
    return p + 1 <= 8


def time_cpu_case(kind, d, p, g, n, fp32, U, n_threads):
    """Seconds for the CPU oracle over elements [0, n): the compiled reference on n_threads
    threads, or (outside the reference's domain, or without it) the C restatement on one."""
    import oracle as O
    import numpy as np
    if kind == "reference" and ref_supports(d, p):
        t, _ = O.ref_time_oracle_mt(d, p, n, g, fp32, U, 1.0 / 1600.0, 2.5, 1.0, (1.0, 1.0, 1.0), False, n_threads)
        return t
    out = np.zeros_like(U)
    ta = time.perf_counter()
    O.oracle_divergence_elements(d, p, g, U, out, 1.0 / 1600.0, 2.5, 1.0, (1.0, 1.0, 1.0), False, 0, n)
    return time.perf_counter() - ta


def cpu_baseline(args, n_threads=None, budget_points=None):
    """The reference oracle (oracle/_ref) on the host cores, bounded sample; returns the cpu_baseline dict."""
    import oracle as O
    if n_threads is None or n_threads <= 0:
        n_threads = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    if budget_points is None:  # ~10 s of reference CPU work at ~4e5 points/s/thread, capped for host memory
        budget_points = min(3e7, 10.0 * 4e5 * (n_threads if kind == "reference" else 1))
    if kind != "reference":
        n_threads = 1
    tot_pts, tot_s, ported = 0, 0.0, []
    for (d, p, precn, g, n) in cpu_sample_cases(args, budget_points):
        fp32 = precn == "fp32"
        U = O.random_field(d, p, n, g, fp32, 2024)
        tot_s += time_cpu_case(kind, d, p, g, n, fp32, U, n_threads)
        tot_pts += n * (p + 1) ** d
        if kind == "reference" and not ref_supports(d, p):
            ported.append(f"d{d} p{p}")
    note = (f"; {', '.join(ported)} lie outside the reference's domain (m <= 8, operators.hpp:18) and were "
            "timed with the C restatement on one thread") if ported else ""
    return {"value": round(tot_pts / tot_s / 1e9, 6), "unit": "GDoF/s", "cores": n_threads, "kind": kind,
            "sample": f"{tot_pts} points across every case of {args.workload} (group-aligned element prefixes, "
                      f"seed 2024), hexfuse::oracle_divergence -O3 on {n_threads} threads, "
                      f"{tot_s:.1f} s of CPU work{note}", "seconds": round(tot_s, 3)}


def run_reference(args, rank):
    if rank != 0:
        return
    import oracle as O
    n_threads = args.cpu_threads if args.cpu_threads and args.cpu_threads > 0 else (os.cpu_count() or 1)
    # size each step so the whole --steps K --warmup W run does ~3e7 points of reference CPU work
    per_step = max(2e5, 3e7 / max(1, args.steps + args.warmup))
    samples = cpu_sample_cases(args, per_step)
    kind = "reference" if O.ref_available() else "port"
    fields = [(d, p, precn, g, n, O.random_field(d, p, n, g, precn == "fp32", 2024)) for (d, p, precn, g, n) in samples]

    def one_step():
        pts, secs = 0, 0.0
        for (d, p, precn, g, n, U) in fields:
            secs += time_cpu_case(kind, d, p, g, n, precn == "fp32", U, n_threads)
            pts += n * (p + 1) ** d
        return pts, secs

    for _ in range(args.warmup):
        one_step()
    P, S = 0, 0.0
    for _ in range(args.steps):
        a, b = one_step()
        P += a
        S += b
    value = P / S / 1e9
    line = {"impl": "reference", "metric": "GDoF/s (solution-point updates/sec), fused flux+divergence; "
                                           "roofline = fraction of HBM",
            "value": round(value, 6), "unit": "GDoF/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(S / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic mt19937_64 uniform(-1,1) fields (random_field, oracle.hpp:154-166)",
            "config": {"workload": args.workload, "description": WORKLOAD_DESC[args.workload],
                       "sample_points_per_step": int(P / args.steps)},
            "cpu_baseline": {"value": round(value, 6), "unit": "GDoF/s", "cores": n_threads, "kind": kind,
                             "sample": f"{int(P / args.steps)} points per step across every case of "
                                       f"{args.workload}, hexfuse::oracle_divergence (reference headers, -O3)"},
            "e2e": {"value": round(value, 6), "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-threads", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
