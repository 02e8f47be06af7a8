#!/bin/bash
# Round 2: tile-mode calibration (every one-chunk variant per caller group) + ncu of four tile kernels.
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python tools/tile_probe.py --d 3 > $O/tile_probe_d3.jsonl 2> $O/tile_probe_d3.err; echo "probe rc=$?"
for spec in "3 fp64 32 7" "3 fp64 32 0" "5 fp32 16 0" "1 fp64 24 1"; do
  set -- $spec
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 2 -c 1 -o $O/tile_p$1_$2_g$3_v$4 \
    python tools/prof_one.py --d 3 --p $1 --prec $2 --group $3 --variant $4 --launches 3 > $O/tile_p$1_$2_g$3_v$4.log 2>&1
  python tools/ncu_brief.py $O/tile_p$1_$2_g$3_v$4.ncu-rep > $O/tile_p$1_$2_g$3_v$4.brief 2>&1
  ncu -i $O/tile_p$1_$2_g$3_v$4.ncu-rep --page raw --csv > $O/tile_p$1_$2_g$3_v$4.raw.csv 2>/dev/null
  rm -f $O/tile_p$1_$2_g$3_v$4.ncu-rep
done
echo done
