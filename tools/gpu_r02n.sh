#!/bin/bash
O=gpurun_out/r02n; mkdir -p $O
timeout 900 python tools/group_sweep.py --d 3 --groups 3,5,15 > $O/groups_odd_d3.jsonl 2> $O/groups_odd.err; echo "sweep rc=$?"
timeout 600 python tools/group_sweep.py --d 2 --groups 3,7,15 > $O/groups_odd_d2.jsonl 2>> $O/groups_odd.err; echo "sweep2 rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "caller_groups or groups_fp64 or misaligned" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
