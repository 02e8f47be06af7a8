#!/bin/bash
# FR right-hand side: one-pass vs two-kernel residual under sustained load (HF_FR_FUSED=1 / 0),
# alternating processes, d = 3 and 2
O=gpurun_out/fr_sus; mkdir -p $O
for r in 1 2; do
  for f in 1 0; do
    HF_FR_FUSED=$f timeout 900 python tools/bench_fr.py --dims 3,2 --sustained 0.5 --out $O/f$f-$r.jsonl > /dev/null 2> $O/f$f-$r.err; echo "f$f-$r rc=$?"
  done
done
