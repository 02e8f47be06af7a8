#!/bin/bash
# Round 2: tile mode, TMA tensor copies vs cp.async 16-byte pieces (HF_TILE=lsu), same box.
O=gpurun_out/r02l; mkdir -p $O
HF_TILE=lsu timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "caller_groups or misaligned" > $O/pytest_lsu.log 2>&1; echo "pytest lsu rc=$?"; tail -1 $O/pytest_lsu.log
for m in tma lsu; do
  HF_TILE=$m PROBE_TAG=$m timeout 900 python tools/tile_probe.py --d 3 --groups 12,20,32,64 > $O/tile_probe_$m.jsonl 2> $O/tile_probe_$m.err; echo "probe $m rc=$?"
done
