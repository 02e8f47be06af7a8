#!/bin/bash
# A/B of the minimum bulk-copy piece (HF_MIN_PIECE) over all lines variants and orders.
O=gpurun_out/abp; mkdir -p $O
for P in ${PIECES:-2048 4096 8192 65536}; do
  [ -f abtest/p$P/libhexfuse_b200.so ] || continue
  HEXFUSE_B200_LIB=$PWD/abtest/p$P/libhexfuse_b200.so timeout 1200 python tools/select_methods.py --dims 3,2 --no-planar --no-unfused --points 1e7 --out $O/sel_p$P.jsonl > /dev/null 2> $O/sel_p$P.err
  echo "p$P rc=$?"
done
