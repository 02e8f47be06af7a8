#!/bin/bash
# FR stages: GPU parity (FR + peer tests), the timing sweep and ncu of the correction kernel (two cases).
O=gpurun_out/${1:-fr}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fr.py tests/test_gpu_peer.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 600 python tools/bench_fr.py --out $O/bench_fr.jsonl > /dev/null 2> $O/bench_fr.err; echo "fr rc=$?"
for c in "2 fp32" "6 fp64"; do
  set -- $c
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:hf_fr_correct -c 1 \
    -o $O/corr_p$1_$2 python tools/prof_fr.py $1 $2 > /dev/null 2>&1; echo "ncu p$1 $2 rc=$?"
done
