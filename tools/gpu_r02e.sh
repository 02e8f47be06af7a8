#!/bin/bash
# Round 2: same-box A/B of the production kernels (pre-tile library lib_alt vs current),
# grouped chunks after the accumulator-layout fix, the staged unfused comparator.
O=gpurun_out/r02e; mkdir -p $O
for i in 1 2; do
  HEXFUSE_B200_LIB=paper_2107_14027_b200/lib_alt/libhexfuse_b200.so timeout 300 python bench.py --no-cpu --no-e2e --no-parity --steps 30 > $O/ab_old_$i.json 2>$O/ab_old_$i.err
  timeout 300 python bench.py --no-cpu --no-e2e --no-parity --steps 30 > $O/ab_new_$i.json 2>$O/ab_new_$i.err
done
echo ab done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "caller_groups or unfused or nonunit" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 600 python tools/group_sweep.py --d 3 --groups 1,2,4,8 > $O/groups_small_d3.jsonl 2> $O/groups_small_d3.err; echo "sweep rc=$?"
timeout 300 python bench.py --workload config4 --no-cpu --no-e2e > $O/bench_config4.json 2> $O/bench_config4.err; echo "c4 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/ncu_config4.csv python bench.py --workload config4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1; echo "ncu rc=$?"
