#!/bin/bash
# executed instructions per launch of candidate kernels (tuning build): fewer SM cycles per
# byte keep a kernel at the roofline when the SM clock drops under a power cap
O=gpurun_out/inst; mkdir -p $O
export HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.avg,smsp__warps_active.avg.per_cycle_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum
for spec in "3 3 fp64 7" "3 3 fp64 0" "3 3 fp64 1" "3 3 fp64 11" "3 3 fp64 19" "3 3 fp64 20" "3 3 fp64 2" \
            "3 6 fp64 3" "3 6 fp64 0" "3 6 fp64 23" "3 3 fp32 7" "3 3 fp32 1" "3 3 fp32 22" "3 5 fp64 1" "3 5 fp64 20"; do
  set -- $spec
  timeout 300 ncu --metrics $M --clock-control none --csv -k regex:hf_lines -c 1 -s 1 python tools/prof_one.py --d $1 --p $2 --prec $3 --variant $4 --launches 2 > $O/d$1p$2$3v$4.csv 2>&1
done
echo done
