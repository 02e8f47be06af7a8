#!/bin/bash
O=gpurun_out/r02x; mkdir -p $O
HF_MAPPED_CS=1 timeout 900 python -m pytest tests/test_gpu_mapped.py -q -x > $O/pytest_cs.log 2>&1; echo "pytest cs rc=$?"; tail -1 $O/pytest_cs.log
for m in 0 1; do HF_MAPPED_CS=$m timeout 900 python tools/bench_mapped.py --dims 3,2 --out $O/bench_mapped_cs$m.jsonl > /dev/null 2> $O/bench_mapped_cs$m.err; echo "mapped $m rc=$?"; done
