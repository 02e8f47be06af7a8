#!/bin/bash
# Round 2: the fused FR residual (stage 1, then ONE kernel for stages 2+3+6+4+5): FR / peer tests,
# and the FR bench with the fused form vs the previous pair (HF_FR_FUSED=0).
O=gpurun_out/r02r; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fr.py tests/test_gpu_peer.py -q -x > $O/pytest_fr.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_fr.log
for m in 1 0; do HF_FR_FUSED=$m timeout 900 python tools/bench_fr.py --out $O/bench_fr_fused$m.jsonl > /dev/null 2> $O/bench_fr_fused$m.err; echo "fr$m rc=$?"; done
