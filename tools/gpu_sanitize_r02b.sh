#!/bin/bash
# compute-sanitizer over the final library's new paths: grouped chunks, the cp.async guarded path,
# the component-split kernel (selected at d3 p4 FP64), PDL chains, CUDA-graph replay.
O=gpurun_out/san_r02b; mkdir -p $O
CS=compute-sanitizer
K1='caller_groups or component_split or dependent_back_to_back or cuda_graph or misaligned or groups_fp64'
timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "$K1" > $O/memcheck.log 2>&1; echo "mem rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "component_split or dependent_back_to_back or caller_groups_d2" > $O/racecheck.log 2>&1; echo "race rc=$?"
timeout 2400 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "component_split or caller_groups_d2" > $O/synccheck.log 2>&1; echo "sync rc=$?"
timeout 1200 $CS --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -k "caller_groups_d2 or misaligned" > $O/initcheck.log 2>&1; echo "init rc=$?"
for f in $O/*.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
