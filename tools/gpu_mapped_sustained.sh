#!/bin/bash
# mapped kernel chunk budget under sustained load: production vs HF_MAPPED_KB=64 / 32 builds,
# alternating processes (A B C A B C), each case 0.6 s back to back
O=gpurun_out/mapped_sus; mkdir -p $O
for r in 1 2; do
  for v in prod kb64 kb32; do
    case $v in prod) L=lib;; *) L=lib_$v;; esac
    HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/$L/libhexfuse_b200.so timeout 900 python tools/bench_mapped.py --sustained 0.6 --out $O/$v$r.jsonl > /dev/null 2> $O/$v$r.err; echo "$v$r rc=$?"
  done
done
