#!/bin/bash
# config-1 bench A/B on one box: current library (d3 p3 FP64 -> variant 26) vs lib_alt (-> 25)
O=gpurun_out/c1ab; mkdir -p $O
sed 's/(3, 3, "fp64"): 4/(3, 3, "fp64"): 2/' bench.py > bench_alt.py
for r in 1 2 3; do
  timeout 300 python bench.py --workload config1 --no-cpu --no-e2e > $O/new$r.json 2>/dev/null
  HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_alt/libhexfuse_b200.so timeout 300 python bench_alt.py --workload config1 --no-cpu --no-e2e > $O/alt$r.json 2>/dev/null
done
for f in $O/*.json; do python -c "import json,sys; r=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', r['value'], r['roofline']['kernel'], r['roofline']['frac'], r['roofline']['step_aggregate_frac'], r['clocks']['sm_mhz'])"; done
