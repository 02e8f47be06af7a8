#!/bin/bash
# compute-sanitizer over FR stage 1 fused on padded chunks (FACES + XP) and the sustained-load selection
O=gpurun_out/san_r02e; mkdir -p $O
CS=compute-sanitizer
K="fused_stage1 or divergence_faces"
timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K" > $O/memcheck.log 2>&1; echo "mem rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K" > $O/racecheck.log 2>&1; echo "race rc=$?"
timeout 2400 $CS --tool synccheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K" > $O/synccheck.log 2>&1; echo "sync rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "padded_chunks or lines_d2" > $O/racecheck_sel.log 2>&1; echo "race sel rc=$?"
for f in $O/*.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
