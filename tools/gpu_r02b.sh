#!/bin/bash
# Round 2: full GPU suite (tile mode, FR interface flux), caller-group sweep.
O=gpurun_out/r02b; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python tools/group_sweep.py --d 3 > $O/groups_d3.jsonl 2> $O/groups_d3.err; echo "sweep3 rc=$?"
timeout 600 python tools/group_sweep.py --d 2 --groups 8,12,16,24,32,40,64 > $O/groups_d2.jsonl 2> $O/groups_d2.err; echo "sweep2 rc=$?"
