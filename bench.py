"""Benchmark driver for the B200 fused flux + divergence kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config2|config1|config3|config4|config5]
                    [--impl ours|reference] [--scaling weak|strong] [--no-e2e] [--no-cpu] [--no-parity]

Metric (BASELINE.json): GDoF/s = solution-point updates per second (all n_v
variables of a point = one update), with the fraction of the HBM roofline of
the dominant kernel (algorithmic bytes = n_v words read + n_v words written
per point, io_model Fused23, io_model.hpp:35).

Default workload = BASELINE config 2, the single-GPU case the metric is quoted
on: d=3 hexes, p = 1..6, FP32 and FP64, ~1e7 solution points per (p,
precision).  One step = one fused launch per (p, precision) = 12 launches over
resident synthetic inputs (uniform(-1,1), every case's input larger than L2).

Multi-GPU: one process per GPU.  Under torchrun (WORLD_SIZE set) each rank owns
its element slice (no data-path collective; NCCL is used only for the barrier,
the max-over-ranks of the device time and the sum of the points).  Without
torchrun, ``--gpus N`` (N > 1) re-launches this script under
``torch.distributed.run`` with N ranks on 127.0.0.1.  `value` is the whole-job
aggregate.  ``--scaling weak`` (default): every rank runs the full per-case
problem; ``--scaling strong``: the case's elements are split across the ranks
(hf_partition, contiguous whole AoSoA groups).

After timing, every rank checks a sample of element groups of every case
against the CPU oracle (test infrastructure, outside the timed region): the
first and last group of the field and 30 more spread over it, so the largest
byte offsets of config 5 (> 4 GB) are covered.  The line carries the worst
relative error per precision (`parity`).

`--impl reference` times the reference's own CPU implementation
(hexfuse::oracle_divergence from /root/reference/proj/include, compiled by
oracle/Makefile into oracle/_ref; the -O3 -march=x86-64-v4/-v3 timing build the
host supports) on all host threads for a bounded sample of the same workload.
That arm never imports the B200 package or touches CUDA: the AoSoA groups come
from the static GPU_GROUPS table below (checked against the library by
tests/test_gpu_scale.py).  Rank 0 alone runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
PARITY_GROUPS = 32
METRIC = "GDoF/s (solution-point updates/sec), fused flux+divergence; roofline = fraction of HBM"

# hf_preferred_group() of the library for every (d, p, precision) a workload uses: the
# AoSoA group that makes one group one kernel chunk.  Static so that the reference arm
# can lay its sample out exactly like the GPU's field without loading the B200 library;
# tests/test_gpu_scale.py checks it against the library.
GPU_GROUPS = {
    (3, 1, "fp32"): 16, (3, 2, "fp32"): 16, (3, 3, "fp32"): 8, (3, 4, "fp32"): 4, (3, 5, "fp32"): 2,
    (3, 6, "fp32"): 4,
    (3, 1, "fp64"): 64, (3, 2, "fp64"): 8, (3, 3, "fp64"): 4, (3, 4, "fp64"): 2, (3, 5, "fp64"): 1,
    (3, 6, "fp64"): 2,
    (2, 1, "fp32"): 64, (2, 2, "fp32"): 64, (2, 3, "fp32"): 64, (2, 4, "fp32"): 32, (2, 5, "fp32"): 8,
    (2, 6, "fp32"): 16, (2, 7, "fp32"): 4, (2, 8, "fp32"): 8,
}


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
    "config5": "d3 hex p=3 and p=5 fp64, 1.5e8 points per case (BASELINE config 5)",
}


def case_elements(d, p, precn, target):
    """(group, whole-problem element count) of one workload case: target points rounded
    to whole groups."""
    g = GPU_GROUPS[(d, p, precn)]
    npt = (p + 1) ** d
    return g, max(g, int(round(target / npt / g)) * g)


def workload_config(workload: str, world: int, scaling: str) -> dict:
    """The `config` object of the JSON line -- identical for both arms (no device state)."""
    pts = 0
    for (d, p, precn, target) in workload_cases(workload):
        _, n = case_elements(d, p, precn, target)
        pts += n * (p + 1) ** d
    if world > 1 and scaling == "weak":
        pts *= world
    return {"workload": workload, "description": WORKLOAD_DESC[workload],
            "cases": len(workload_cases(workload)), "points_per_step": pts,
            "l2": "no flush; every case's input+output exceeds the 126 MB L2",
            "parallelism": f"element-partition x{world} ({scaling if world > 1 else 'single GPU'})"}


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
    """Samples SM clock + throttle reasons through NVML every ~1 ms while running (short timed
    regions -- config 1 is ~7 ms for both passes -- still get several samples)."""

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
            time.sleep(0.001)

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


# ------------------------------------------------------------------------------------------------ ranks
class Ranks:
    """rank / world / local rank and the three reductions the bench needs.  NCCL
    reduces device tensors, gloo (the CPU self-test) host tensors."""

    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.gpu = self.local
        self.dev = None

    def init(self, backend: str, device=None):
        self.dev = device
        if self.world > 1:
            import torch.distributed as dist
            kw = {"device_id": device} if backend == "nccl" else {}
            dist.init_process_group(backend, **kw)

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def _reduce(self, x: float, op: str) -> float:
        if self.world == 1:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=getattr(dist.ReduceOp, op))
        return float(t.item())

    def max(self, x: float) -> float:
        return self._reduce(x, "MAX")

    def sum(self, x: float) -> float:
        return self._reduce(x, "SUM")


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun: re-launch under torch.distributed.run, one rank
    per GPU on this node; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------------------------------------ ours
def launches_per_call(info: dict, n_elem: int, group: int, word_bytes: int, total_words: int) -> int:
    """Kernel launches of one hf_fused_divergence call: the TMA-ring variant runs the full
    chunks persistently and the partial / allocation-final chunk in a second launch
    (hf_launch.cuh launch_lines_pipe)."""
    if not info["name"].startswith("hf_lines_pipe"):
        return 1
    ne = info["elems_per_cta"]
    n_full = n_elem // ne
    if group == ne and n_full > 0 and n_full * ne == n_elem and (total_words * word_bytes) % 16:
        n_full -= 1
    return 1 + (1 if n_full < -(-n_elem // ne) else 0)


def parity_sample(hf, cases, rank, n_groups_sample):
    """Checker (outside the timed region): the fused result of sampled element groups of every
    case against the CPU oracle (oracle_divergence restated, oracle.hpp:20-62).  Returns the
    per-case worst relative error (verify.hpp:19-33 definition over the sampled elements)."""
    import numpy as np

    import oracle as O
    out = []
    for ci, c in enumerate(cases):
        d, p, g = c["d"], c["p"], c["group"]
        nv, npt = 1 + d + d * d, (p + 1) ** d
        gw = g * npt * nv
        n_groups = -(-c["n_elem"] // g)
        rng = np.random.default_rng(7919 * (rank + 1) + ci)
        pick = {0, n_groups - 1}
        if n_groups > 2:
            pick |= set(int(x) for x in rng.choice(np.arange(1, n_groups - 1),
                                                   size=min(n_groups - 2, n_groups_sample - 2), replace=False))
        maxdiff, maxref = 0.0, 0.0
        for gi in sorted(pick):
            n_e = min(g, c["n_elem"] - gi * g)
            U = c["u"][gi * gw:(gi + 1) * gw].double().cpu().numpy()
            got = c["o"][gi * gw:(gi + 1) * gw].double().cpu().numpy()
            ref = O.oracle_divergence(d, p, n_e, g, U, 1.0 / 1600.0, 2.5, 1.0)
            real = (np.arange(g) < n_e)[None, None, :]
            a = got.reshape(nv, npt, g)
            b = ref.reshape(nv, npt, g)
            diff = np.where(real, np.abs(a - b), 0.0)
            if not np.all(np.isfinite(diff)):
                maxdiff = float("inf")
            maxdiff = max(maxdiff, float(diff.max()))
            maxref = max(maxref, float(np.where(real, np.abs(b), 0.0).max()))
        out.append({"groups": len(pick), "last_byte_offset": (n_groups * gw) * c["u"].element_size(),
                    "max_rel_err": maxdiff / max(1.0, maxref)})
    return out


def run_ours(args, R: Ranks):
    import torch

    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import PhysParams, Precision

    rank, world = R.rank, R.world
    local_rank = R.gpu  # the rank's GPU (its local rank; 0 for every rank with HF_BENCH_SHARED_GPU)
    dev = torch.device("cuda", local_rank)
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    peak, peak_src = load_peaks()
    traffic = load_traffic()
    st = torch.cuda.current_stream()

    # ---- allocate every case's resident input/output on this rank
    cases = []
    gen = torch.Generator(device=dev)
    gen.manual_seed(2024 + rank)
    launches = 0
    for (d, p, precn, target) in workload_cases(args.workload):
        prec = Precision[precn]
        g, n_total = case_elements(d, p, precn, target)
        lib_g = hf.preferred_group(hf.make_problem(d, p, 1, 1, prec, par))
        if lib_g != g:
            raise SystemExit(f"bench.py GPU_GROUPS[{(d, p, precn)}] = {g} but the library prefers {lib_g}")
        npt = (p + 1) ** d
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
        launches += launches_per_call(info, n_elem, g, wb, words)
        cases.append({"d": d, "p": p, "precision": precn, "pr": pr, "u": u, "o": o, "n_elem": n_elem,
                      "points": n_elem * npt, "alg_bytes": n_elem * npt * 2 * hf.n_vars(d) * wb,
                      "kernel": info["name"], "group": g, "info": info})
        assert u.numel() * wb * 2 > L2_BYTES or args.workload == "config3", "input must exceed L2"

    def step():
        for c in cases:
            hf.fused_divergence_device(c["pr"], c["u"], c["o"], st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- per-launch durations for the roofline, just before the timed region: every case K
    # times, in blocks of ROOF_BLOCK launches back to back between one CUDA-event pair on the
    # launching stream (inside a block consecutive launches overlap launch and ramp-up as in
    # the timed region), the blocks round-robin over the cases so that every case sees the
    # same mix of clock and thermal state
    ROOF_BLOCK = 5
    blocks = [(c_i, min(ROOF_BLOCK, args.steps - k0)) for k0 in range(0, args.steps, ROOF_BLOCK)
              for c_i in range(len(cases))]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in blocks]
    # ---- timed region (value): K steps (a step = every case once) launched back to back with
    # one event pair around all of them -- consecutive launches overlap launch and ramp-up with
    # the previous kernel's tail (programmatic dependent launch, hf_launch.cuh launch_kernel)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        R.barrier()
        torch.cuda.synchronize()
        for (c_i, reps), (a, b) in zip(blocks, ev):
            c = cases[c_i]
            a.record(st)
            for _ in range(reps):
                hf.fused_divergence_device(c["pr"], c["u"], c["o"], st)
            b.record(st)
        torch.cuda.synchronize()
        R.barrier()
        torch.cuda.synchronize()
        t0.record(st)
        for k in range(args.steps):
            step()
        t1.record(st)
        torch.cuda.synchronize()
        R.barrier()
    elapsed = R.max(t0.elapsed_time(t1) * 1e-3)
    # A timed region of a few milliseconds (config 1) fits one or two NVML samples: the same
    # step is then repeated for ~0.3 s, untimed, with a second sampler -- the clocks the
    # workload runs at under sustained load, reported beside the in-region ones.
    clk_sustained = None
    if len(clk.samples) < 5:
        with ClockSampler(local_rank) as clk2:
            t_end = time.perf_counter() + 0.3
            while time.perf_counter() < t_end:
                for _ in range(10):
                    step()
                torch.cuda.synchronize()
        clk_sustained = clk2.summary()
    per_case = [0.0] * len(cases)
    for (c_i, reps), (a, b) in zip(blocks, ev):
        per_case[c_i] += a.elapsed_time(b) * 1e-3 / args.steps
    points_rank = sum(c["points"] for c in cases)
    points_all = R.sum(points_rank)
    value = points_all * args.steps / elapsed / 1e9

    # ---- per-case roofline, dominant kernel
    case_rows = []
    for c, tavg in zip(cases, per_case):
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
        R.barrier()
        ta = time.perf_counter()
        for _ in range(e2e_steps):
            ctx.run_batch(batch)
        tb = time.perf_counter()
        R.barrier()
        te = R.max(tb - ta)
        pts_e = R.sum(sum(h[3] for h in hosts))
        h2d = sum(h[0].numel() * h[0].element_size() for h in hosts)
        e2e = {"value": round(pts_e * e2e_steps / te / 1e9, 4), "unit": "GDoF/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d, "steps": e2e_steps,
               "path": "hf_fused_divergence_host_batch (pinned host buffers, one 3-stream slice pipeline per step)"}
        if frac < 1.0:
            e2e["sample"] = f"each case cut to {frac:.3f} of its elements (host RAM {host_ram / 2**30:.0f} GiB)"
        # the e2e result must equal the device-resident run's result
        same = all(torch.equal(h[1].to(dev), c["o"][: h[1].numel()]) for h, c in zip(hosts, cases))
        e2e["matches_device_result"] = bool(R.sum(0.0 if same else 1.0) == 0.0)
        ctx.close()
        del hosts

    # ---- unfused comparator beside it (config 4)
    unfused = None
    if args.workload == "config4":
        # the unfused comparator (io_model S2 + S3, io_model.hpp:32-33) on the same problem in
        # its own AoSoA group (hf_preferred_group of HF_METHOD_UNFUSED), same points
        c = cases[0]
        from paper_2107_14027_b200 import Method
        pr_u0 = hf.make_problem(c["d"], c["p"], 1, 1, c["pr"].precision, par, method=Method.unfused)
        gu = hf.preferred_group(pr_u0)
        nu_el = max(gu, c["n_elem"] // gu * gu)
        pr_u = hf.make_problem(c["d"], c["p"], nu_el, gu, c["pr"].precision, par, method=Method.unfused)
        uu = torch.empty(hf.field_words(pr_u), dtype=c["u"].dtype, device=dev).uniform_(-1.0, 1.0, generator=gen)
        ou = torch.empty_like(uu)
        ws = torch.empty(hf.unfused_workspace_bytes(pr_u) // uu.element_size(), dtype=uu.dtype, device=dev)
        for _ in range(3):
            hf.unfused_divergence_device(pr_u, uu, ou, ws, st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.steps):
            hf.unfused_divergence_device(pr_u, uu, ou, ws, st)
        b.record(st)
        torch.cuda.synchronize()
        tu = a.elapsed_time(b) * 1e-3 / args.steps
        upts = nu_el * (c["p"] + 1) ** c["d"]
        ubpp = 8 * hf.n_vars(c["d"]) * uu.element_size()
        tf = case_rows[0]["us_per_launch"] * 1e-6 / c["points"] * upts  # fused time for the same points
        unfused = {"kernels": hf.kernel_info(pr_u)["name"], "group": gu, "points": upts,
                   "us_per_step": round(tu * 1e6, 2), "gdofs": round(upts / tu / 1e9, 3),
                   "alg_bytes_per_point": ubpp, "achieved_GBps": round(upts * ubpp / tu / 1e9, 1),
                   "frac": round(upts * ubpp / tu / 1e9 / peak, 4),
                   "fused_speedup": round(tu / tf, 3), "model_speedup": 4.0}
        del uu, ou, ws

    # ---- parity (checker, after timing): sampled groups of every case against the CPU oracle
    parity = None
    if not args.no_parity:
        rows = parity_sample(hf, cases, rank, PARITY_GROUPS)
        worst = {}
        for c, r, cr in zip(cases, rows, case_rows):
            cr["parity_rel_err"] = float(f"{r['max_rel_err']:.3e}")
            worst[c["precision"]] = max(worst.get(c["precision"], 0.0), r["max_rel_err"])
        worst = {k: R.max(v) for k, v in sorted(worst.items())}
        tol = {"fp32": 1e-5, "fp64": 1e-12}
        parity = {"max_rel_err": {k: float(f"{v:.3e}") for k, v in worst.items()},
                  "tol": {k: tol[k] for k in worst}, "ok": all(v <= tol[k] for k, v in worst.items()),
                  "groups_per_case": min(PARITY_GROUPS, min(r["groups"] for r in rows)),
                  "max_byte_offset": max(r["last_byte_offset"] for r in rows),
                  "oracle": "oracle_divergence (oracle.hpp:20-62) restated in oracle/hexfuse_oracle.c, "
                            "first + last + 30 random element groups per case and rank"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, n_threads=args.cpu_threads)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 4), "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps * 1e3, 4),
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32+f64" if args.workload in ("config2",) else
            ("f64" if all(c["precision"] == "fp64" for c in cases) else "f32"),
            "data": "synthetic uniform(-1,1) fields, resident in HBM",
            "config": workload_config(args.workload, world, args.scaling),
            "method": "auto (measured selection table)",
            "roofline": roofline, "cases": case_rows, "e2e": e2e, "parity": parity, "cpu_baseline": cpu,
            "gpu_launches": args.steps * launches, "gpu_launches_roofline_pass": args.steps * launches,
            "timing": "value: K steps back to back between one CUDA-event pair (max over ranks); roofline and "
                      "cases: just before it, each case K times in blocks of 5 back-to-back launches between "
                      "an event pair, the blocks round-robin over the cases",
            "clocks": clk.summary(),
            **({"clocks_sustained": clk_sustained} if clk_sustained else {}),
        }
        if unfused:
            line["unfused"] = unfused
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------ reference CPU
def cpu_sample_cases(workload: str, budget_points: float):
    """Bounded, group-aligned sample of every case of the workload (same d, p, precision and
    AoSoA group as the GPU's field), each case's share proportional to its points in the
    GPU workload."""
    cases = workload_cases(workload)
    sizes = [case_elements(d, p, precn, t)[1] * (p + 1) ** d for (d, p, precn, t) in cases]
    tot = float(sum(sizes))
    out = []
    for (d, p, precn, _), sz in zip(cases, sizes):
        g = GPU_GROUPS[(d, p, precn)]
        npt = (p + 1) ** d
        n = max(g, int(budget_points * sz / tot / npt) // g * g)
        out.append((d, p, precn, g, n))
    return out


def ref_supports(d, p):
    """The reference oracle's domain: gauss_legendre_points accepts m <= 8 (operators.hpp:18)."""
    return p + 1 <= 8


def cpu_threads(requested):
    import oracle as O
    return requested if requested and requested > 0 else O.host_cpu()["logical_cpus"]


def time_cpu_case(kind, d, p, g, n, fp32, U, n_threads):
    """Seconds for the CPU oracle over elements [0, n): the reference's timing build on n_threads
    threads, or (outside the reference's domain, or without it) the C restatement on one."""
    import numpy as np

    import oracle as O
    if kind == "reference" and ref_supports(d, p):
        t, _ = O.ref_time_oracle_mt(d, p, n, g, fp32, U, 1.0 / 1600.0, 2.5, 1.0, (1.0, 1.0, 1.0), False, n_threads,
                                    timing_build=True)
        return t
    out = np.zeros_like(U)
    ta = time.perf_counter()
    O.oracle_divergence_elements(d, p, g, U, out, 1.0 / 1600.0, 2.5, 1.0, (1.0, 1.0, 1.0), False, 0, n)
    return time.perf_counter() - ta


def sample_field(kind, d, p, n, g, fp32):
    import oracle as O
    if kind == "reference" and ref_supports(d, p):
        return O.ref_random_field_timing(d, p, n, g, fp32, 2024)  # hexfuse::random_field, oracle.hpp:154-166
    return O.random_field(d, p, n, g, fp32, 2024)


def cpu_kind():
    import oracle as O
    try:
        O.ref_timing()
        return "reference"
    except Exception:
        return "port"


def cpu_desc(kind, n_threads):
    import oracle as O
    hc = O.host_cpu()
    build = O.ref_timing()[1] if kind == "reference" else "C restatement -O2 (1 thread)"
    return hc, build


def cpu_baseline(args, n_threads=None, budget_points=None):
    """The reference oracle (oracle/_ref) on the host cores, bounded sample; returns the cpu_baseline dict."""
    kind = cpu_kind()
    n_threads = cpu_threads(n_threads) if kind == "reference" else 1
    if budget_points is None:  # ~10 s of reference CPU work at ~4e5 points/s/thread, capped for host memory
        budget_points = min(3e7, 10.0 * 4e5 * n_threads)
    tot_pts, tot_s, ported = 0, 0.0, []
    for (d, p, precn, g, n) in cpu_sample_cases(args.workload, budget_points):
        fp32 = precn == "fp32"
        U = sample_field(kind, d, p, n, g, fp32)
        tot_s += time_cpu_case(kind, d, p, g, n, fp32, U, n_threads)
        tot_pts += n * (p + 1) ** d
        if kind == "reference" and not ref_supports(d, p):
            ported.append(f"d{d} p{p}")
    hc, build = cpu_desc(kind, n_threads)
    note = (f"; {', '.join(ported)} lie outside the reference's domain (m <= 8, operators.hpp:18) and were "
            "timed with the C restatement on one thread") if ported else ""
    return {"value": round(tot_pts / tot_s / 1e9, 6), "unit": "GDoF/s", "cores": n_threads, "kind": kind,
            "cpu_model": hc["model"], "host_logical_cpus": hc["logical_cpus"], "build": build,
            "sample": f"{tot_pts} points across every case of {args.workload} (group-aligned element prefixes "
                      f"in the GPU's AoSoA groups, each case's share proportional to its points, seed 2024), "
                      f"hexfuse::oracle_divergence {build} on {n_threads} threads, {tot_s:.1f} s of CPU work{note}",
            "seconds": round(tot_s, 3)}


def run_reference(args, R: Ranks):
    """The reference arm: rank 0 alone; no B200 package, no CUDA."""
    if R.rank != 0:
        return
    kind = cpu_kind()
    n_threads = cpu_threads(args.cpu_threads) if kind == "reference" else 1
    # size each step so the whole --steps K --warmup W run does --ref-budget points of reference CPU work (~8 s)
    per_step = max(2e4, args.ref_budget / max(1, args.steps + args.warmup))
    samples = cpu_sample_cases(args.workload, per_step)
    fields = [(d, p, precn, g, n, sample_field(kind, d, p, n, g, precn == "fp32")) for (d, p, precn, g, n) in samples]

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
    hc, build = cpu_desc(kind, n_threads)
    line = {"impl": "reference", "metric": METRIC,
            "value": round(value, 6), "unit": "GDoF/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(S / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": args.scaling if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic mt19937_64 uniform(-1,1) fields (hexfuse::random_field, oracle.hpp:154-166)",
            "config": workload_config(args.workload, args.gpus, args.scaling),
            "cpu_baseline": {"value": round(value, 6), "unit": "GDoF/s", "cores": n_threads, "kind": kind,
                             "cpu_model": hc["model"], "host_logical_cpus": hc["logical_cpus"], "build": build,
                             "sample": f"{int(P / args.steps)} points per step across every case of "
                                       f"{args.workload} (the GPU's AoSoA groups, each case's share proportional "
                                       f"to its points), hexfuse::oracle_divergence ({build}) on {n_threads} "
                                       "threads, one contiguous group-aligned sub-field per thread"},
            "e2e": {"value": round(value, 6), "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------ self-test
def run_selftest(args, R: Ranks):
    """CPU self-test of the multi-rank plumbing (HF_BENCH_SELFTEST=1, gloo): the launch, the
    barriers and the max / sum reductions of the real run, with every rank's device work
    replaced by a sleep of (rank + 1) * 10 ms per step.  Prints a line marked "selftest"."""
    per_rank_points = 1000 * (R.rank + 1)
    R.barrier()
    ta = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.01 * (R.rank + 1))
    own = time.perf_counter() - ta
    R.barrier()
    elapsed = R.max(own)
    pts = R.sum(per_rank_points)
    if R.rank == 0:
        print(json.dumps({"selftest": True, "metric": METRIC, "value": pts * args.steps / elapsed / 1e9,
                          "unit": "GDoF/s", "n_gpus": R.world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": elapsed / args.steps * 1e3, "rank0_ms_per_step": own / args.steps * 1e3,
                          "points_all": pts, "config": workload_config(args.workload, R.world, args.scaling)}),
              flush=True)


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
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--ref-budget", type=float, default=1e8, help="reference arm: points of CPU work per run")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    R = Ranks()
    selftest = os.environ.get("HF_BENCH_SELFTEST") == "1"
    if args.impl == "reference":
        run_reference(args, R)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args.gpus))
    if selftest:
        R.init("gloo")
        try:
            run_selftest(args, R)
        finally:
            R.close()
        return
    import torch
    if os.environ.get("HF_BENCH_SHARED_GPU") == "1":
        # functional test of the N-rank path on a one-GPU box: every rank on GPU 0, the
        # bench's scalar reductions over gloo (timings then share the GPU -- not a bench number)
        R.gpu = 0
        torch.cuda.set_device(0)
        R.init("gloo")
    else:
        if R.world > 1 and torch.cuda.device_count() < R.world:
            raise SystemExit(f"bench.py: {R.world} ranks but {torch.cuda.device_count()} visible GPUs")
        torch.cuda.set_device(R.local)
        R.init("nccl", torch.device("cuda", R.local))
    try:
        run_ours(args, R)
    finally:
        R.close()


if __name__ == "__main__":
    main()
