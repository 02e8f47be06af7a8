#!/bin/bash
# Round 2: grouped chunks + calibrated tile choice: GPU suite, default bench (production kernels
# must not regress), caller-group sweep d3/d2.
O=gpurun_out/r02d; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
timeout 900 python tools/group_sweep.py --d 3 --groups 1,2,4,8,12,15,16,20,24,32,40,64 > $O/groups_d3.jsonl 2> $O/groups_d3.err; echo "sweep3 rc=$?"
timeout 600 python tools/group_sweep.py --d 2 --groups 1,2,4,8,12,16,24,32,40,64 > $O/groups_d2.jsonl 2> $O/groups_d2.err; echo "sweep2 rc=$?"
