#!/bin/bash
# compute-sanitizer over the padded x-row chunks (lines variants 25-27, TMA-padded staging)
O=gpurun_out/san_r02d; mkdir -p $O
CS=compute-sanitizer
K="lines_variants and (25 or 26 or 27)"
timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" > $O/memcheck.log 2>&1; echo "mem rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" > $O/racecheck.log 2>&1; echo "race rc=$?"
timeout 2400 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" > $O/synccheck.log 2>&1; echo "sync rc=$?"
timeout 1200 $CS --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" > $O/initcheck.log 2>&1; echo "init rc=$?"
for f in $O/*.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
