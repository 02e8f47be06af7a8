#!/bin/bash
O=gpurun_out/r02v; mkdir -p $O
HF_TILE_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "caller_groups" > $O/pytest_split.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_split.log
for m in 0 1; do HF_TILE_SPLIT=$m timeout 900 python tools/tile_probe.py --d 3 --groups 12,24,32,64 > $O/tile_split$m.jsonl 2> $O/tile_split$m.err; echo "probe $m rc=$?"; done
