#!/bin/bash
# ncu --set full with source counters for the weakest selected kernels (one launch each).
mkdir -p gpurun_out/prof
run() { # tag d p prec variant
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 1 -c 1 \
    -o gpurun_out/prof/$1 python tools/prof_one.py --d $2 --p $3 --prec $4 --variant $5 --launches 2 > gpurun_out/prof/$1.log 2>&1
  ncu -i gpurun_out/prof/$1.ncu-rep --page source --csv > gpurun_out/prof/$1_src.csv 2>/dev/null
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/$1.ncu-rep --page details --csv > gpurun_out/prof/$1_details.csv 2>/dev/null
}
run p6f32v3 3 6 fp32 3
run p6f64v3 3 6 fp64 3
run p4f32v5 3 4 fp32 5
run d2p2f32v3 2 2 fp32 3
run d2p1f32v0 2 1 fp32 0
mkdir -p gpurun_out/prof_keep; rm -f gpurun_out/prof/*.ncu-rep
ls -la gpurun_out/prof
