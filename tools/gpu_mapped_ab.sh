#!/bin/bash
# mapped kernel A/B on one box: production (SPLIT=1) vs lib_alt (EXTRA=-DHF_MAPPED_SPLIT=2)
O=gpurun_out/mapped_ab; mkdir -p $O
HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_alt/libhexfuse_b200.so timeout 900 python -m pytest tests/test_gpu_mapped.py -q -x > $O/pytest_alt.log 2>&1; tail -1 $O/pytest_alt.log
for v in prod alt prod2 alt2; do
  case $v in prod*) L=lib;; alt*) L=lib_alt;; esac
  HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/$L/libhexfuse_b200.so timeout 900 python tools/bench_mapped.py --out $O/$v.jsonl > /dev/null 2> $O/$v.err; echo "$v rc=$?"
done
