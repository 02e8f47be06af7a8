#!/bin/bash
O=gpurun_out/r02w; mkdir -p $O
for spec in "3 3 fp64" "3 6 fp32" "3 1 fp32"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:hf_mapped -s 1 -c 1 -o $O/mapped_p$2_$3 \
    python tools/prof_mapped.py --d $1 --p $2 --prec $3 > $O/mapped_p$2_$3.log 2>&1
  python tools/ncu_brief.py $O/mapped_p$2_$3.ncu-rep > $O/mapped_p$2_$3_brief.txt 2>&1
  ncu -i $O/mapped_p$2_$3.ncu-rep --page source --csv > $O/mapped_p$2_$3_src.csv 2>/dev/null
  python tools/ncu_src_top.py $O/mapped_p$2_$3_src.csv > $O/mapped_p$2_$3_srctop.txt 2>&1
  ncu -i $O/mapped_p$2_$3.ncu-rep --page raw --csv > $O/mapped_p$2_$3_raw.csv 2>/dev/null
  rm -f $O/mapped_p$2_$3.ncu-rep $O/mapped_p$2_$3_src.csv
done
timeout 600 python tools/bench_mapped.py --dims 3 --out $O/bench_mapped.jsonl > /dev/null 2>&1; echo mapped rc=$?
