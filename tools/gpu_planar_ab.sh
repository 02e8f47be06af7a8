#!/bin/bash
# planar register cap A/B: production vs HF_PLANAR_REGS=128 (lib_alt) vs 96 (lib_alt2), same box
O=gpurun_out/planar_ab; mkdir -p $O
for v in prod alt alt2; do
  if [ $v = prod ]; then L=lib; else L=lib_$v; fi
  HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/$L/libhexfuse_b200.so timeout 900 python tools/select_methods.py --dims 3 --ps 1,2,3 --variants 0 --no-unfused --points 1e7 --out $O/$v.jsonl > /dev/null 2> $O/$v.err
  echo "$v rc=$?"
done
