"""Launch the FR right-hand side of one (p, precision) on a ~1e7-point periodic
mesh twice: a short command to put under ncu (kernels hf_fr_project / hf_fr_correct)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2107_14027_b200 as hf  # noqa: E402
from paper_2107_14027_b200 import PhysParams, Precision  # noqa: E402

p, prec = int(sys.argv[1]), Precision[sys.argv[2]]
par = PhysParams(1 / 1600, 2.5, 1.0)
g = hf.preferred_group(hf.make_problem(3, p, 1, 1, prec, par))
m = p + 1
nx = ny = 16
while (nx * ny) % g:
    nx += 1
nz = max(2, int(1e7 / m ** 3 / (nx * ny)))
dims = (nx, ny, nz)
n = nx * ny * nz
pr = hf.make_problem(3, p, n, g, prec, par)
dt = torch.float32 if prec == Precision.fp32 else torch.float64
u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda")
uf = torch.empty(hf.face_words(pr), dtype=dt, device="cuda")
out = torch.empty_like(u)
for _ in range(2):
    hf.fr_residual_device(pr, dims, u, uf, out)
torch.cuda.synchronize()
