#!/bin/bash
# ncu --set full with source counters of the p6 TMA-ring kernels (FP64, FP32)
O=gpurun_out/prof_ring; mkdir -p $O
for spec in "fp64" "fp32"; do
  out=$O/p6$spec
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 1 -c 1 -o $out \
    python tools/prof_one.py --d 3 --p 6 --prec $spec --variant 3 --launches 2 > $out.log 2>&1
  ncu -i $out.ncu-rep --page source --csv > ${out}_src.csv 2>/dev/null
  python tools/ncu_brief.py $out.ncu-rep > ${out}_brief.txt 2>&1
  python tools/ncu_src_top.py ${out}_src.csv > ${out}_srctop.txt 2>&1
  rm -f $out.ncu-rep
done
echo done
