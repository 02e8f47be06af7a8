#!/bin/bash
# A/B ncu captures of one lines variant: abtest/lib_base.so vs the tuning build.
# usage: tools/gpu_prof_ab.sh "d p prec variant" ...
O=gpurun_out/profab; mkdir -p $O
for spec in "$@"; do
  set -- $spec
  for tag in base:abtest/lib_base.so cur:paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so; do
    name=${tag%%:*}; lib=${tag#*:}
    out=$O/d$1p$2$3v$4_$name
    HEXFUSE_B200_LIB=$PWD/$lib timeout 300 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 1 -c 1 \
      -o $out python tools/prof_one.py --d $1 --p $2 --prec $3 --variant $4 --launches 2 > $out.log 2>&1
    ncu -i $out.ncu-rep --page raw --csv > ${out}_raw.csv 2>/dev/null
    ncu -i $out.ncu-rep --page source --csv > ${out}_src.csv 2>/dev/null
    rm -f $out.ncu-rep
  done
done
ls $O
