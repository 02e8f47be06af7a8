"""Probe: does recording CUDA events between launches change a kernel's time?
30 back-to-back launches timed as a whole vs 30 launches each bracketed by events."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

par = PhysParams(1 / 1600, 2.5, 1.0)
for p, prec, v in [(6, Precision.fp32, 1), (6, Precision.fp32, 3), (3, Precision.fp64, 7), (6, Precision.fp64, 3),
                   (6, Precision.fp64, 0)]:
    pr0 = hf.make_problem(3, p, 1, 1, prec, par)
    try:
        g = hf.variant_info(pr0, Method.lines, v)["elems_per_cta"]
    except Exception as e:
        print(p, prec.name, v, e)
        continue
    n = int(round(1e7 / (p + 1) ** 3 / g)) * g
    pr = hf.make_problem(3, p, n, g, prec, par)
    dt = torch.float32 if prec == Precision.fp32 else torch.float64
    u = torch.rand(hf.field_words(pr), dtype=dt, device='cuda') * 2 - 1
    o = torch.empty_like(u)
    f = lambda: hf.fused_divergence_variant(pr, Method.lines, v, u, o)  # noqa: E731
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30):
        f()
    b.record()
    b.synchronize()
    t_block = a.elapsed_time(b) / 30 * 1e3
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
    a.record()
    for e0, e1 in evs:
        e0.record()
        f()
        e1.record()
    b.record()
    b.synchronize()
    t_ev_total = a.elapsed_time(b) / 30 * 1e3
    t_ev_each = sum(e0.elapsed_time(e1) for e0, e1 in evs) / 30 * 1e3
    name = hf.variant_info(pr, Method.lines, v)["name"]
    print(f"{name}: no events {t_block:.1f} us | with events: total {t_ev_total:.1f} us, per-launch {t_ev_each:.1f} us",
          flush=True)
