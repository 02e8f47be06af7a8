"""CUDA-graph replay of the fused launches vs stream launches (same box, same buffers).

For config 1 (one case) and config 2 (12 cases): time K steps launched on a stream back to
back, and the same K steps captured once into a CUDA graph (torch.cuda.CUDAGraph) and
replayed -- the launches keep their programmatic-dependent-launch attribute inside the
graph.  Checks that the replayed results equal the stream-launched ones bit for bit.

    python tools/graph_probe.py > profiles/r02/graph_probe.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402

PAR = PhysParams(1.0 / 1600.0, 2.5, 1.0)


def cases_of(workload):
    out = []
    for (d, p, precn, target) in bench.workload_cases(workload):
        g, n = bench.case_elements(d, p, precn, target)
        prec = Precision[precn]
        pr = hf.make_problem(d, p, n, g, prec, PAR)
        dt = torch.float32 if prec == Precision.fp32 else torch.float64
        u = torch.empty(hf.field_words(pr), dtype=dt, device="cuda").uniform_(-1, 1)
        out.append((pr, u, torch.empty_like(u), n * (p + 1) ** d))
    return out


def main():
    K = 20
    for workload in ("config1", "config2", "config3"):
        cs = cases_of(workload)
        st = torch.cuda.Stream()
        torch.cuda.synchronize()

        def step():
            for pr, u, o, _ in cs:
                hf.fused_divergence_device(pr, u, o, st)
        with torch.cuda.stream(st):
            for _ in range(3):
                step()
        torch.cuda.synchronize()
        ref = [o.clone() for _, _, o, _ in cs]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(K):
            step()
        b.record(st)
        b.synchronize()
        t_stream = a.elapsed_time(b) * 1e-3 / K
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(K):
                step()
        for o in (x[2] for x in cs):
            o.zero_()
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize()
        same = all(torch.equal(o, r) for (_, _, o, _), r in zip(cs, ref))
        with torch.cuda.stream(st):  # replay() launches on the current stream
            g.replay()
            a.record(st)
            g.replay()
            b.record(st)
        b.synchronize()
        t_graph = a.elapsed_time(b) * 1e-3 / K
        pts = sum(c[3] for c in cs)
        print(json.dumps({"workload": workload, "cases": len(cs), "steps": K,
                          "stream_ms_per_step": round(t_stream * 1e3, 4), "graph_ms_per_step": round(t_graph * 1e3, 4),
                          "stream_gdofs": round(pts / t_stream / 1e9, 3), "graph_gdofs": round(pts / t_graph / 1e9, 3),
                          "graph_equals_stream": same}), flush=True)
        del cs, ref, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
