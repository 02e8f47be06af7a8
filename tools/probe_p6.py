"""Probe: one kernel timed (a) back-to-back on the same buffers, (b) alternating with
another case's kernel, (c) rotating over two buffer sets -- per-launch CUDA events."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import Method, PhysParams, Precision  # noqa: E402

par = PhysParams(1 / 1600, 2.5, 1.0)


def case(p, prec, variant=None):
    g = hf.preferred_group(hf.make_problem(3, p, 1, 1, prec, par)) if variant is None else \
        hf.variant_info(hf.make_problem(3, p, 1, 1, prec, par), Method.lines, variant)["elems_per_cta"]
    n = int(round(1e7 / (p + 1) ** 3 / g)) * g
    pr = hf.make_problem(3, p, n, g, prec, par)
    dt = torch.float32 if prec == Precision.fp32 else torch.float64
    u = torch.rand(hf.field_words(pr), dtype=dt, device='cuda') * 2 - 1
    o = torch.empty_like(u)
    w = 4 if prec == Precision.fp32 else 8
    name = hf.kernel_info(pr)['name'] if variant is None else hf.variant_info(pr, Method.lines, variant)['name']
    fn = (lambda: hf.fused_divergence_device(pr, u, o)) if variant is None else \
        (lambda: hf.fused_divergence_variant(pr, Method.lines, variant, u, o))
    return fn, n * (p + 1) ** 3 * 2 * 13 * w, name


def per_launch(seq, reps=20):
    """seq: list of (fn, bytes, name); returns mean us per entry over reps rounds."""
    for _ in range(3):
        for f, _, _ in seq:
            f()
    torch.cuda.synchronize()
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in seq] for _ in range(reps)]
    for r in range(reps):
        for i, (f, _, _) in enumerate(seq):
            evs[r][i][0].record()
            f()
            evs[r][i][1].record()
    torch.cuda.synchronize()
    return [sum(evs[r][i][0].elapsed_time(evs[r][i][1]) for r in range(reps)) / reps * 1e3 for i in range(len(seq))]


A = case(6, Precision.fp32)
A2 = case(6, Precision.fp32)
B = case(5, Precision.fp32)
C = case(6, Precision.fp64)
V3 = case(6, Precision.fp32, variant=3)
for label, seq in [("same buffers", [A]), ("two buffer sets", [A, A2]), ("after p5 fp32", [B, A]),
                   ("after p6 fp64", [C, A]), ("pipe v3 after p5", [B, V3]), ("pipe v3 alone", [V3])]:
    ts = per_launch(seq)
    print(label, " | ".join(f"{s[2]} {t:.1f} us {s[1] / t / 1e3:.0f} GB/s" for s, t in zip(seq, ts)), flush=True)
