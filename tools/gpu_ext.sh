#!/bin/bash
# Extensions: GPU parity of the mapped-element and FR-stage kernels,
# their timing sweeps, and one ncu capture of each new kernel.
O=gpurun_out/ext; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fr.py tests/test_gpu_mapped.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 900 python tools/bench_mapped.py --dims 3 --out $O/bench_mapped.jsonl > /dev/null 2> $O/bench_mapped.err; echo "mapped rc=$?"
timeout 900 python tools/bench_fr.py --out $O/bench_fr.jsonl > /dev/null 2> $O/bench_fr.err; echo "fr rc=$?"
cat > $O/prof_fr.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2107_14027_b200 as hf
from paper_2107_14027_b200 import PhysParams, Precision
p = int(sys.argv[1]); prec = Precision[sys.argv[2]]
par = PhysParams(1/1600, 2.5, 1.0)
g = hf.preferred_group(hf.make_problem(3, p, 1, 1, prec, par))
m = p + 1
nx = ny = 16
while (nx * ny) % g: nx += 1
nz = max(2, int(1e7 / m**3 / (nx * ny)))
dims = (nx, ny, nz); n = nx * ny * nz
pr = hf.make_problem(3, p, n, g, prec, par)
dt = torch.float32 if prec == Precision.fp32 else torch.float64
u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda")
uf = torch.empty(hf.face_words(pr), dtype=dt, device="cuda"); out = torch.empty_like(u)
for _ in range(2):
    hf.fr_residual_device(pr, dims, u, uf, out)
torch.cuda.synchronize()
PY
for k in hf_fr_project hf_fr_correct; do
  out=$O/ncu_${k}_p3fp64
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o $out python $O/prof_fr.py 3 fp64 > $out.log 2>&1
  ncu -i $out.ncu-rep --page details --csv > ${out}_details.csv 2>/dev/null
  ncu -i $out.ncu-rep --page source --csv > ${out}_src.csv 2>/dev/null
  rm -f $out.ncu-rep
done
echo done
