#!/bin/bash
# ncu --set full of the FR correction kernel (stages 4+5) for a few (p, precision) cases.
O=gpurun_out/proffr; mkdir -p $O
for c in "2 fp32" "6 fp64" "6 fp32" "4 fp64"; do
  set -- $c
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:hf_fr_correct -c 1 \
    -o $O/corr_p$1_$2 python tools/prof_fr.py $1 $2 > $O/corr_p$1_$2.log 2>&1; echo "p$1 $2 rc=$?"
done
