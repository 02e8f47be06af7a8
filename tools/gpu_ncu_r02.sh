#!/bin/bash
# ncu launch list of the default bench (final library) -> profiles/ncu_traffic.json, plus full captures of
# the two slowest config-2 kernels.
O=gpurun_out/ncu_r02; mkdir -p $O
timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file $O/ncu_launches_config2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_bench.json 2>&1
echo "ncu list rc=$?"
python tools/ncu_traffic.py $O/ncu_launches_config2.csv $O/bench_config2.json $O/ncu_traffic.json 3 > $O/ncu_traffic.txt 2>&1; echo "traffic rc=$?"
for spec in "6 fp64 -1" "6 fp32 -1" "4 fp64 -1"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 1 -c 1 -o $O/full_p$1_$2 \
    python tools/prof_one.py --d 3 --p $1 --prec $2 --variant $3 --launches 2 > $O/full_p$1_$2.log 2>&1
  python tools/ncu_brief.py $O/full_p$1_$2.ncu-rep > $O/full_p$1_$2_brief.txt 2>&1
  rm -f $O/full_p$1_$2.ncu-rep
done
echo done
