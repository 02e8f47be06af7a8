#!/bin/bash
# FR one-pass residual on padded chunks: parity, then compute-sanitizer
O=gpurun_out/san_r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fr.py tests/test_gpu_peer.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
CS=compute-sanitizer
K="residual"
timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K" > $O/memcheck.log 2>&1; echo "mem rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K" > $O/racecheck.log 2>&1; echo "race rc=$?"
timeout 2400 $CS --tool synccheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K" > $O/synccheck.log 2>&1; echo "sync rc=$?"
for f in $O/*check.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
