#!/bin/bash
# tile ring (lines variant 24): full GPU suite, then the caller-group sweep at d3 p5
mkdir -p gpurun_out/tilering
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tilering/pytest.log 2>&1; tail -3 gpurun_out/tilering/pytest.log
timeout 600 python tools/group_sweep.py --d 3 --ps 5 --groups 4,8,12,16,20,24,32,40,64 > gpurun_out/tilering/groups_p5.jsonl 2> gpurun_out/tilering/groups.err; echo "sweep rc=$?"; tail -2 gpurun_out/tilering/groups.err
