#!/bin/bash
# ncu --set full of the planar kernel (method a) at p2 FP32 and p3 FP64
O=gpurun_out/prof_planar; mkdir -p $O
for spec in "2 fp32" "3 fp64"; do
  set -- $spec
  out=$O/planar_p$1_$2
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:hf_planar -s 1 -c 1 -o $out \
    python tools/prof_one.py --d 3 --p $1 --prec $2 --method planar --launches 2 > $out.log 2>&1
  python tools/ncu_brief.py $out.ncu-rep > ${out}_brief.txt 2>&1
  ncu -i $out.ncu-rep --page source --csv > ${out}_src.csv 2>/dev/null
  python tools/ncu_src_top.py ${out}_src.csv > ${out}_srctop.txt 2>&1
  ncu -i $out.ncu-rep --page details --csv > ${out}_details.csv 2>/dev/null
  rm -f $out.ncu-rep
done
echo done
