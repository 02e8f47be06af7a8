#!/bin/bash
# Mapped-element kernel: GPU parity, timing sweep beside the constant-Jacobian kernel, one ncu capture.
O=gpurun_out/${OUT:-mapped}; mkdir -p $O
SPECS=${SPECS:-"3 3 fp64;3 6 fp64"}
if [ -z "$PROF_ONLY" ]; then
timeout 600 python -m pytest tests/test_gpu_mapped.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 900 python tools/bench_mapped.py --out $O/bench_mapped.jsonl > /dev/null 2> $O/bench_mapped.err; echo "bench rc=$?"
fi
cat > $O/prof.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2107_14027_b200 as hf
from paper_2107_14027_b200 import PhysParams, Precision
d, p, prec = int(sys.argv[1]), int(sys.argv[2]), Precision[sys.argv[3]]
par = PhysParams(1/1600, 2.5, 1.0)
g = hf.mapped_kernel_info(hf.make_problem(d, p, 1, 1, prec, par))["elems_per_cta"]
n = int(1e7 / (p + 1) ** d) // g * g
pr = hf.make_problem(d, p, n, g, prec, par)
dt = torch.float32 if prec == Precision.fp32 else torch.float64
u = torch.rand(hf.field_words(pr), dtype=dt, device="cuda")
geo = torch.rand(hf.geometry_words(pr), dtype=dt, device="cuda") * 0.1
gv = geo.view(-1, 1 << d, d, g)
for c in range(1 << d):
    for x in range(d):
        gv[:, c, x] += 0.5 if (c >> x) & 1 else -0.5
o = torch.empty_like(u)
for _ in range(2):
    hf.fused_divergence_mapped_device(pr, u, geo, o)
torch.cuda.synchronize()
PY
IFS=";" read -ra SPL <<< "$SPECS"
for spec in "${SPL[@]}"; do
  set -- $spec
  out=$O/ncu_d$1p$2$3
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:hf_mapped -s 1 -c 1 -o $out python $O/prof.py $1 $2 $3 > $out.log 2>&1
  ncu -i $out.ncu-rep --page raw --csv > ${out}_raw.csv 2>/dev/null
  ncu -i $out.ncu-rep --page source --csv > ${out}_src.csv 2>/dev/null
  ncu -i $out.ncu-rep --page details --csv > ${out}_details.csv 2>/dev/null
done
echo done
